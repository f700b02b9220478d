mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
MST_TAIL_TRACE=1 python tools/mst_once.py --config c1 --warmup 1 --reps 1
for t in 1.2e7 6e6; do for c in c1 c0 c2; do echo -n "tail=$t "; MST_TAIL_EDGES=$t python tools/mst_once.py --config $c --warmup 3 --reps 20 | head -1; done; done
for c in c1 c0 c2 c3; do echo -n "nodedup "; MST_TAIL_DEDUP=0 python tools/mst_once.py --config $c --warmup 3 --reps 10 | head -1; done
python tools/mst_once.py --config c3 --warmup 2 --reps 5
python tools/mst_once.py --config c4 --warmup 1 --reps 3
} > gpurun_out/exp2.log 2>&1
