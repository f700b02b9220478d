mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
CONFIGS="c1 c4" REPS=10 bash tools/ab.sh; cat gpurun_out/ab.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp8_c1_launches.csv python tools/mst_once.py --config c1 --warmup 1 --reps 1 > /dev/null 2>&1
} > gpurun_out/exp8.log 2>&1
