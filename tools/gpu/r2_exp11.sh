set -x
mkdir -p gpurun_out/exp11
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 2 --reps 5 | head -1; }
{ for C in c3 c4 c2; do run MST_RETIRE=1; run MST_RETIRE=0; run MST_RETIRE=1; run MST_RETIRE=0; done; } > gpurun_out/exp11/sweep.txt 2>&1
grep -v "^+" gpurun_out/exp11/sweep.txt
MST_TIMELINE=1 MST_DEBUG_ROUNDS=1 python tools/mst_once.py --config c3 --warmup 1 --reps 1 > gpurun_out/exp11/c3_r1.txt 2>&1
