set -x
mkdir -p gpurun_out/exp17
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 2 --reps 5 | head -1; }
{ for C in c4 c3 c2; do run MST_GIANT_LIGHT=0; run MST_GIANT_LIGHT=1; run MST_GIANT_LIGHT=1 MST_GIANT_BITS=1e6; run MST_GIANT_LIGHT=0 MST_GIANT_BITS=1e6; done; } > gpurun_out/exp17/sweep.txt 2>&1
grep -v "^+" gpurun_out/exp17/sweep.txt
