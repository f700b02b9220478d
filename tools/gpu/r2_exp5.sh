# light-phase retirement: parity first, then A/B
set -x
mkdir -p gpurun_out/exp5
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp5/tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/exp5/tests.log
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 2 --reps 5 | head -1; }
{
for C in c4 c2 c3; do
run MST_RETIRE=1
run MST_RETIRE=0
run MST_RETIRE=1 MST_FILTER_BETA=1.0
run MST_RETIRE=1 MST_FILTER_BETA=1.25
run MST_RETIRE=1 MST_FILTER_BETA=2.0
done
} > gpurun_out/exp5/sweep.txt 2>&1
grep -v "^+" gpurun_out/exp5/sweep.txt
MST_DEBUG_ROUNDS=1 MST_TIMELINE=1 python tools/mst_once.py --config c4 --warmup 1 --reps 1 > gpurun_out/exp5/c4_timeline.txt 2>&1
tail -80 gpurun_out/exp5/c4_timeline.txt | grep -v "^timeline.*k_scan" | tail -70
