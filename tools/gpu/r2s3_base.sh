# round 2 session 3: re-entry baseline
set -x
mkdir -p gpurun_out/s3base
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s3base/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3base/tests.log
for C in c4 c3 c2 c1 c0; do echo -n "$C: "; timeout 300 python tools/mst_once.py --config $C --warmup 3 --reps 10 | head -1; done
MST_TIMELINE=1 timeout 300 python tools/mst_once.py --config c4 --warmup 1 --reps 1 > gpurun_out/s3base/timeline_c4.txt 2>&1
MST_TIMELINE=1 timeout 300 python tools/mst_once.py --config c1 --warmup 1 --reps 1 > gpurun_out/s3base/timeline_c1.txt 2>&1
