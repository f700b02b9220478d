# Filter-Boruvka light-set size sweep (MST_FILTER_BETA: light edges ~ beta * n)
mkdir -p gpurun_out
{
for c in ${CONFIGS:-c4 c3 c2 c0}; do
  for b in ${BETAS:-1 1.5 2 3 4}; do
    echo -n "$c beta=$b: "; MST_FILTER_BETA=$b timeout 300 python tools/mst_once.py --config $c --warmup 2 --reps ${REPS:-5} | head -1
  done
done
} > gpurun_out/sweep_beta.log 2>&1
