# sparse emit A/B + tests
mkdir -p gpurun_out/s3e6
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 3 --reps 10 | head -1; }
{ for C in c4 c3; do run MST_EMIT_SPARSE=0; run MST_EMIT_SPARSE=1; run MST_EMIT_SPARSE=0; run MST_EMIT_SPARSE=1; done; } > gpurun_out/s3e6/sweep.txt 2>&1
cat gpurun_out/s3e6/sweep.txt
MST_TIMELINE=1 timeout 300 python tools/mst_once.py --config c4 --warmup 1 --reps 1 > gpurun_out/s3e6/timeline_c4.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3e6/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3e6/tests.log
