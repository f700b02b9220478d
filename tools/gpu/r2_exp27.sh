set -x
mkdir -p gpurun_out/exp27
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 3 --reps 10 | head -1; }
{ for C in c4; do for mb in 128 160 192 256 384 600; do run MST_RANGE_MB=$mb; done; run MST_RANGE_OFFERS=0; done; for C in c3 c2; do for mb in 64 128 192; do run MST_RANGE_MB=$mb; done; run MST_RANGE_OFFERS=0; done; } > gpurun_out/exp27/sweep.txt 2>&1
grep "^c[0-9]\|^MST" gpurun_out/exp27/sweep.txt
for mb in 128 192; do MST_RANGE_MB=$mb MST_TIMELINE=1 python tools/mst_once.py --config c4 --warmup 1 --reps 1 > gpurun_out/exp27/timeline_c4_$mb.txt 2>&1; done
