mkdir -p gpurun_out
bash tools/round_bench.sh
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python tools/mst_once.py --config c1 --warmup 1 --reps 1 > gpurun_out/ncu_c1.log 2>&1; echo "ncu rc=$?"
for c in c1 c2 c3 c4; do python tools/mst_once.py --config $c --warmup 2 --reps 5; done > gpurun_out/once.log 2>&1
