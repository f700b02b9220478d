mkdir -p gpurun_out
{
timeout 1400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/sanitize.py 2>&1 | tail -1
for rep in 1 2; do for t in 1 0; do for c in c1 c0; do echo -n "start_c=$t "; MST_TAIL_START_C=$t python tools/mst_once.py --config $c --warmup 3 --reps 20 | head -1; done; done; done
MST_TAIL_TRACE=1 python tools/mst_once.py --config c1 --warmup 1 --reps 1 2>&1 | head -1
} > gpurun_out/exp_start_c.log 2>&1
