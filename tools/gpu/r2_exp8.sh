set -x
mkdir -p gpurun_out/exp8
for v in 0 1; do MST_RETIRE=$v MST_DEBUG_ROUNDS=1 MST_TIMELINE=1 python tools/mst_once.py --config c3 --warmup 1 --reps 1 > gpurun_out/exp8/c3_r$v.txt 2>&1; done
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 2 --reps 10 | head -1; }
{ for C in c0 c1; do run MST_X=0; run MST_X=0; done; } > gpurun_out/exp8/small.txt 2>&1
grep -v "^+" gpurun_out/exp8/small.txt
