set -x
mkdir -p gpurun_out/exp24
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp24/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp24/tests.log
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 3 --reps 10 | head -1; }
{ for C in c4 c3 c2; do run MST_X=0; run MST_X=0; done; } > gpurun_out/exp24/sweep.txt 2>&1
grep -v "^+" gpurun_out/exp24/sweep.txt
MST_TIMELINE=1 python tools/mst_once.py --config c4 --warmup 1 --reps 1 > gpurun_out/exp24/timeline_c4.txt 2>&1
