mkdir -p gpurun_out
{
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do for lz in 1 0; do echo -n "lazy=$lz "; MST_LAZY_ROUND1=$lz python tools/mst_once.py --config c1 --warmup 3 --reps 10 | head -1; done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp11_c1_launches.csv python tools/mst_once.py --config c1 --warmup 1 --reps 1 > /dev/null 2>&1
} > gpurun_out/exp11.log 2>&1
