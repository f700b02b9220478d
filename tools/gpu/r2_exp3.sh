# offer filter reads through L1 (MST_OFFER_CACHED bitmask of sites: 1 min1, 2 split, 4 count, 8 heavy)
# and the per-launch stream timeline of c1 / c4
set -x
mkdir -p gpurun_out/exp3
for c in c4 c2 c3 c0 c1; do for v in 0 15 0 15; do echo -n "$c OFFER_CACHED=$v "; MST_OFFER_CACHED=$v timeout 300 python tools/mst_once.py --config $c --warmup 2 --reps 5 | head -1; done; done > gpurun_out/exp3/cached.txt 2>&1
for c in c4 c2; do for v in 2 4 8 6 12; do echo -n "$c OFFER_CACHED=$v "; MST_OFFER_CACHED=$v timeout 300 python tools/mst_once.py --config $c --warmup 2 --reps 5 | head -1; done; done >> gpurun_out/exp3/cached.txt 2>&1
cat gpurun_out/exp3/cached.txt
for c in c1 c4 c0; do MST_TIMELINE=1 timeout 300 python tools/mst_once.py --config $c --warmup 2 --reps 1 > gpurun_out/exp3/timeline_$c.txt 2>&1; done
MST_TAIL_TRACE=1 timeout 300 python tools/mst_once.py --config c1 --warmup 2 --reps 1 > gpurun_out/exp3/tailtrace_c1.txt 2>&1
tail -40 gpurun_out/exp3/timeline_c1.txt
