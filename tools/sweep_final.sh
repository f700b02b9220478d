# last knob sweep on the final code: tail CTAs/SM, small-n tail entry
mkdir -p gpurun_out
{
for c in c1 c0 c2 c3; do
  for v in "" MST_TAIL_BPS=1 MST_TAIL_SMALL_N=262144 MST_TAIL_SMALL_N=16384; do
    echo -n "$c ${v:-base}: "; env $v timeout 300 python tools/mst_once.py --config $c --warmup 3 --reps 10 | head -1
  done
done
} > gpurun_out/sweep_final.log 2>&1
