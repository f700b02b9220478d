# MST_TAIL_EDGES x MST_DEDUP_MIN_EDGES sweep (device-resident ms/MST, mst_once)
mkdir -p gpurun_out
for c in ${CONFIGS:-c1 c0 c2}; do
  for t in ${TAILS:-3e6 1e6 3e5 1e5}; do
    for d in ${DEDUPS:-2e6}; do
      echo -n "$c tail=$t dedup_min=$d: "
      MST_TAIL_EDGES=$t MST_DEDUP_MIN_EDGES=$d timeout 120 python tools/mst_once.py --config $c --warmup 3 --reps 20 | head -1
    done
  done
done 2>&1 | tee gpurun_out/sweep_tail.txt
