# Evidence pass: bench lines for every config, launch list of the bench
# command, one ncu --set full capture of a c1 MST, launch lists of c3/c4.
mkdir -p gpurun_out/prof
cd $GRAFT_REPO_ROOT
for c in c1 c0 c2 c3 c4; do
  timeout 900 python bench.py --config $c > gpurun_out/prof/bench_$c.json 2> gpurun_out/prof/bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/prof/bench_c1_reference.json 2>gpurun_out/prof/ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/bench_c1_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_launch.log 2>&1; echo "launch rc=$?"
ncu --set full --clock-control none --import-source on -f -o gpurun_out/prof/c1_full \
  python tools/mst_once.py --config c1 --warmup 0 --reps 1 > gpurun_out/prof/ncu_full.log 2>&1; echo "full rc=$?"
for c in c3 c4; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof/${c}_launches.csv \
  python tools/mst_once.py --config $c --warmup 0 --reps 1 > gpurun_out/prof/ncu_$c.log 2>&1; echo "$c launches rc=$?"
done
