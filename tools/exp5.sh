mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c1 c0 c2 c3 c4; do python tools/mst_once.py --config $c --warmup 3 --reps 10 | head -1; done
echo -n "nofilt "; MST_FILTER_TABLE_MB=1 python tools/mst_once.py --config c1 --warmup 3 --reps 10 | head -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp5_c1_launches.csv python tools/mst_once.py --config c1 --warmup 1 --reps 1 > /dev/null 2>&1
} > gpurun_out/exp5.log 2>&1
