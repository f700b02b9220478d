set -x
mkdir -p gpurun_out/exp12
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp12/tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/exp12/tests.log
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 2 --reps 5 | head -1; }
{ for C in c4 c3 c2; do run MST_BUCKET_OFFERS=1; run MST_BUCKET_OFFERS=0; run MST_BUCKET_SHIFT=21; run MST_BUCKET_SHIFT=23; done; } > gpurun_out/exp12/sweep.txt 2>&1
grep -v "^+" gpurun_out/exp12/sweep.txt
MST_TIMELINE=1 MST_DEBUG_ROUNDS=1 python tools/mst_once.py --config c4 --warmup 1 --reps 1 > gpurun_out/exp12/c4.txt 2>&1
