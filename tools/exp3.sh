mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
MST_TAIL_TRACE=1 python tools/mst_once.py --config c1 --warmup 1 --reps 1
for c in c1 c0 c2 c3; do echo -n "dedup "; python tools/mst_once.py --config $c --warmup 3 --reps 10 | head -1; echo -n "nodedup "; MST_TAIL_DEDUP=0 python tools/mst_once.py --config $c --warmup 3 --reps 10 | head -1; done
for r in 2 8; do echo -n "ratio $r "; MST_TAIL_DEDUP_RATIO=$r python tools/mst_once.py --config c1 --warmup 3 --reps 10 | head -1; done
} > gpurun_out/exp3.log 2>&1
