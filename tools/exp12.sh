mkdir -p gpurun_out
{
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/sanitize.py 2>&1 | tail -2
for rep in 1 2; do for lz in 1 0; do echo -n "lazytail=$lz "; MST_LAZY_TAIL=$lz python tools/mst_once.py --config c1 --warmup 3 --reps 10 | head -1; done; done
MST_TAIL_TRACE=1 python tools/mst_once.py --config c1 --warmup 1 --reps 1 2>&1 | head -1
} > gpurun_out/exp12.log 2>&1
