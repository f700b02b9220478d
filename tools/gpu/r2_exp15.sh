set -x
mkdir -p gpurun_out/exp15
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp15/tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/exp15/tests.log
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 3 --reps 20 | head -1; }
{ for C in c1 c0; do run MST_ROUND1_C=1; run MST_ROUND1_C=0; run MST_ROUND1_C=1; run MST_ROUND1_C=0; done; for C in c2 c3 c4; do run MST_X=0; done; } > gpurun_out/exp15/sweep.txt 2>&1
grep -v "^+" gpurun_out/exp15/sweep.txt
for c in c1 c0; do MST_TIMELINE=1 MST_TAIL_TRACE=1 python tools/mst_once.py --config $c --warmup 2 --reps 1 > gpurun_out/exp15/timeline_$c.txt 2>&1; done
tail -12 gpurun_out/exp15/timeline_c1.txt
