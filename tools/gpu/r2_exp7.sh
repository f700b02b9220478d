# heavy filter vertex records: parity, then A/B
set -x
mkdir -p gpurun_out/exp7
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp7/tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/exp7/tests.log
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 2 --reps 5 | head -1; }
{
for C in c4 c2 c3; do
run MST_HEAVY_INFO=1
run MST_HEAVY_INFO=0
run MST_RETIRE=0
for b in 1.0 1.25; do run MST_FILTER_BETA=$b; done
done
} > gpurun_out/exp7/sweep.txt 2>&1
grep -v "^+" gpurun_out/exp7/sweep.txt
MST_DEBUG_ROUNDS=1 MST_TIMELINE=1 python tools/mst_once.py --config c4 --warmup 1 --reps 1 > gpurun_out/exp7/c4_timeline.txt 2>&1
tail -45 gpurun_out/exp7/c4_timeline.txt | grep -v "k_scan"
