set -x
mkdir -p gpurun_out/exp26
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp26/tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/exp26/tests.log
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 3 --reps 10 | head -1; }
{ for C in c4 c3; do run MST_RANGE_OFFERS=1; run MST_RANGE_OFFERS=0; for mb in 32 96 128; do run MST_RANGE_MB=$mb; done; run MST_RANGE_OFFERS=1 MST_OFFER_HEAVY=2 MST_OFFER_SPLIT=2; done; } > gpurun_out/exp26/sweep.txt 2>&1
grep "^c[0-9]\|^MST" gpurun_out/exp26/sweep.txt
MST_TIMELINE=1 python tools/mst_once.py --config c4 --warmup 1 --reps 1 > gpurun_out/exp26/timeline_c4.txt 2>&1
