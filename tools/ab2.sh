mkdir -p gpurun_out
{
for c in c4 c3; do for rep in 1 2; do
echo -n "$c new split1: "; MST_OFFER_SPLIT=1 python tools/mst_once.py --config $c --warmup 3 --reps 5 | head -1
echo -n "$c new split2: "; python tools/mst_once.py --config $c --warmup 3 --reps 5 | head -1
echo -n "$c new notail: "; MST_TAIL=0 python tools/mst_once.py --config $c --warmup 3 --reps 5 | head -1
echo -n "$c old notail: "; MST_GPU_LIB=tools/ab/libmstgpu_dbb66c2.so MST_TAIL=0 python tools/mst_once.py --config $c --warmup 3 --reps 5 | head -1
done; done
} > gpurun_out/ab2.log 2>&1
