mkdir -p gpurun_out
{
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/filter_rule.py
for c in c1 c0 c2 c3 c4; do python tools/mst_once.py --config $c --warmup 3 --reps 5 | head -1; done
} > gpurun_out/exp_small_n.log 2>&1
