mkdir -p gpurun_out
{
for c in c1 c0 c2; do for rep in 1 2; do
echo -n "$c base: "; python tools/mst_once.py --config $c --warmup 3 --reps 10 | head -1
echo -n "$c tail3 bps3: "; MST_GPU_LIB=tools/ab/libmstgpu_tail3.so MST_TAIL_BPS=3 python tools/mst_once.py --config $c --warmup 3 --reps 10 | head -1
echo -n "$c tail4 bps4: "; MST_GPU_LIB=tools/ab/libmstgpu_tail4.so MST_TAIL_BPS=4 python tools/mst_once.py --config $c --warmup 3 --reps 10 | head -1
echo -n "$c tail4 bps2: "; MST_GPU_LIB=tools/ab/libmstgpu_tail4.so MST_TAIL_BPS=2 python tools/mst_once.py --config $c --warmup 3 --reps 10 | head -1
done; done
MST_GPU_LIB=tools/ab/libmstgpu_tail4.so MST_TAIL_BPS=4 MST_TAIL_TRACE=1 python tools/mst_once.py --config c1 --warmup 1 --reps 1 2>&1 | head -2
} > gpurun_out/ab3.log 2>&1
