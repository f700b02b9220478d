set -x
mkdir -p gpurun_out/exp10
for v in 0 1; do MST_RETIRE=$v MST_DEBUG_ROUNDS=1 MST_TIMELINE=1 python tools/mst_once.py --config c3 --warmup 1 --reps 1 > gpurun_out/exp10/c3_r$v.txt 2>&1; done
