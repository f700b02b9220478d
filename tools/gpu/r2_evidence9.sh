# round-2 evidence, pass 9: final build of round 2 (after the L1-cached hot-table reads)
set -x
mkdir -p gpurun_out/ev9
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/ev9/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ev9/tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev9/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/ev9/bench_c4.json 2> gpurun_out/ev9/bench_c4.err; echo "c4 rc=$?"
for c in c0 c1 c2 c3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ev9/bench_$c.json 2> gpurun_out/ev9/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev9/bench_c4_reference.json 2> gpurun_out/ev9/ref.err; echo "ref rc=$?"
for c in c1 c4; do MST_TIMELINE=1 MST_DEBUG_ROUNDS=1 timeout 300 python tools/mst_once.py --config $c --warmup 2 --reps 1 > gpurun_out/ev9/timeline_$c.txt 2>&1; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__m_xbar2l1tex_read_sectors.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
for c in c4 c1; do
timeout 1200 ncu --metrics $M --clock-control none --replay-mode application --csv --log-file gpurun_out/ev9/${c}_launches.csv python tools/mst_once.py --config $c --warmup 0 --reps 1 > gpurun_out/ev9/${c}_launches.log 2>&1; echo "launches $c rc=$?"
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev9/bench_c4_launchlist.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev9/bench_c4_ncu.log 2>&1; echo "bench launch list rc=$?"
du -sh gpurun_out
