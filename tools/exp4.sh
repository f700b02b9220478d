mkdir -p gpurun_out
{
for t in 6e6 2e6 1e6 5e5; do for d in 4 2; do
echo -n "tail=$t div=$d active=1e6 min=1e6: "; MST_TAIL_EDGES=$t MST_DEDUP_ACTIVE=1e6 MST_DEDUP_MIN_EDGES=1e6 MST_DEDUP_TABLE_DIV=$d python tools/mst_once.py --config c1 --warmup 3 --reps 10 | head -2 | tr '\n' ' '; echo
done; done
echo -n "default "; python tools/mst_once.py --config c1 --warmup 3 --reps 10 | head -1
MST_TAIL_TRACE=1 python tools/mst_once.py --config c1 --warmup 1 --reps 1
} > gpurun_out/exp4.log 2>&1
