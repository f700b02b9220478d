set -x
mkdir -p gpurun_out/exp9
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 2 --reps 5 | head -1; }
{ for C in c3 c4 c2; do run MST_RETIRE=1; run MST_RETIRE=0; run MST_RETIRE=1; run MST_RETIRE=0; done; } > gpurun_out/exp9/sweep.txt 2>&1
grep -v "^+" gpurun_out/exp9/sweep.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp9/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp9/tests.log
