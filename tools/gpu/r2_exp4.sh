# light-phase dedup from round 2 with a large pair table; beta re-check with cached offers; parity
set -x
mkdir -p gpurun_out/exp4
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 2 --reps 5 | head -1; }
{
for C in c4 c2 c3; do
run MST_X=0
run MST_DEDUP_ACTIVE=4e6 MST_DEDUP_TABLE_DIV=1 MST_DEDUP_CAP_LOG2=27
run MST_DEDUP_ACTIVE=4e6 MST_DEDUP_TABLE_DIV=2 MST_DEDUP_CAP_LOG2=27
run MST_DEDUP_ACTIVE=4e6 MST_DEDUP_TABLE_DIV=1 MST_DEDUP_CAP_LOG2=26
for b in 1.0 1.25 2.0 3.0; do run MST_FILTER_BETA=$b; done
done
} > gpurun_out/exp4/sweep.txt 2>&1
cat gpurun_out/exp4/sweep.txt
C=c4 MST_DEBUG_ROUNDS=1 MST_DEDUP_ACTIVE=4e6 MST_DEDUP_TABLE_DIV=1 MST_DEDUP_CAP_LOG2=27 python tools/mst_once.py --config c4 --warmup 0 --reps 1 2>&1 | tail -14
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp4/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp4/tests.log
