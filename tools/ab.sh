# A/B: in-tree library vs tools/ab/libmstgpu_*.so on the same box
mkdir -p gpurun_out
{
for c in ${CONFIGS:-c2 c3 c4}; do
  for rep in 1 2; do
    for lib in "" tools/ab/*.so; do
      echo -n "$c ${lib:-new}: "; MST_GPU_LIB=$lib timeout 300 python tools/mst_once.py --config $c --warmup 3 --reps ${REPS:-5} | head -1
    done
  done
done
} > gpurun_out/ab.log 2>&1
