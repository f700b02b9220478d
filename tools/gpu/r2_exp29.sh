set -x
mkdir -p gpurun_out/exp29
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp29/tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/exp29/tests.log
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 3 --reps 10 | head -1; }
{ for C in c4 c3 c2; do run MST_STASH_MB=64; run MST_STASH_MB=0; run MST_STASH_MB=32; run MST_STASH_MB=128; done; } > gpurun_out/exp29/sweep.txt 2>&1
grep "^c[0-9]\|^MST" gpurun_out/exp29/sweep.txt
MST_TIMELINE=1 python tools/mst_once.py --config c4 --warmup 1 --reps 1 > gpurun_out/exp29/timeline_c4.txt 2>&1
