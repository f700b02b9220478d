mkdir -p gpurun_out
{
for f in 1 0; do echo -n "filter=$f "; MST_FILTER=$f python tools/mst_once.py --config c0 --warmup 3 --reps 10 | head -1; done
for t in 3e6 1.5e6 6e6; do echo -n "filter tail=$t "; MST_TAIL_EDGES=$t python tools/mst_once.py --config c0 --warmup 3 --reps 10 | head -1; done
python tools/mst_once.py --config c0 --warmup 1 --reps 1
MST_TAIL_TRACE=1 python tools/mst_once.py --config c0 --warmup 1 --reps 1 2>&1 | head -3
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c0_launches.csv python tools/mst_once.py --config c0 --warmup 0 --reps 1 > /dev/null 2>&1
} > gpurun_out/exp_c0.log 2>&1
