mkdir -p gpurun_out
{
timeout 1400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do for b in 1 0; do for c in c1 c0 c2 c3 c4; do echo -n "bulk=$b "; MST_BULK_COPY=$b python tools/mst_once.py --config $c --warmup 3 --reps 5 | head -1; done; done; done
} > gpurun_out/exp_bulk.log 2>&1
