set -x
mkdir -p gpurun_out/exp28
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp28/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp28/tests.log
for c in c4 c3 c2; do timeout 900 python tools/shard_time.py --config $c --shards 1,2 --reps 2; done > gpurun_out/exp28/shard.txt 2>&1
cat gpurun_out/exp28/shard.txt
