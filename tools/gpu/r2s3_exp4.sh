# lazy-ends split A/B + tests
mkdir -p gpurun_out/s3e4
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 3 --reps 10 | head -1; }
{ for C in c4 c3 c2; do run MST_LAZY_ENDS=0; run MST_LAZY_ENDS=1; run MST_LAZY_ENDS=0; run MST_LAZY_ENDS=1; done; } > gpurun_out/s3e4/sweep.txt 2>&1
cat gpurun_out/s3e4/sweep.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3e4/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3e4/tests.log
