mkdir -p gpurun_out
{
python tools/e2e_breakdown.py --config c1 --reps 4
python tools/e2e_breakdown.py --config c1 --reps 4 --flush
MST_TAIL_TRACE=1 python tools/mst_once.py --config c1 --warmup 1 --reps 1
CONFIGS=c1 TAILS="1.2e7 6e6 3.5e6 2e6 1e6" bash tools/sweep_tail.sh
} > gpurun_out/exp1.log 2>&1
