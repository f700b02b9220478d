mkdir -p gpurun_out
{
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
MST_TAIL_TRACE=1 python tools/mst_once.py --config c1 --warmup 1 --reps 1 2>&1 | head -1
CONFIGS="c1 c0 c2 c3" REPS=10 bash tools/ab.sh; cat gpurun_out/ab.log
} > gpurun_out/exp10.log 2>&1
