# tail entry threshold (MST_TAIL_EDGES overrides both the plain 6e6 and light 3e6 defaults)
mkdir -p gpurun_out
{
for c in c1 c0; do for t in "" 3e6 1e7; do echo -n "$c tail=${t:-default}: "; MST_TAIL_EDGES=$t python tools/mst_once.py --config $c --warmup 3 --reps 10 | head -1; done; done
for c in c2 c3 c4; do for t in "" 1.5e6 6e6; do echo -n "$c tail=${t:-default}: "; MST_TAIL_EDGES=$t python tools/mst_once.py --config $c --warmup 2 --reps 5 | head -1; done; done
} > gpurun_out/sweep_tail2.log 2>&1
