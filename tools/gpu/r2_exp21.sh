set -x
mkdir -p gpurun_out/exp21
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 2 --reps 5 | head -1; }
{ for C in c4 c3 c2; do run MST_X=0; run MST_OFFER_HEAVY=2; run MST_OFFER_SPLIT=2; run MST_OFFER_HEAVY=2 MST_OFFER_SPLIT=2; run MST_OFFER_COUNT=2; run MST_OFFER_HEAVY=0; done; } > gpurun_out/exp21/sweep.txt 2>&1
grep "^c[0-9]\|^MST" gpurun_out/exp21/sweep.txt
