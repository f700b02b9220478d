# per-launch table of one c4 / c1 MST with the L1 miss-path sectors added
mkdir -p gpurun_out/p3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__m_xbar2l1tex_read_sectors.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
for c in c4 c1; do
timeout 1200 ncu --metrics $M --clock-control none --replay-mode application --csv --log-file gpurun_out/p3/${c}_launches.csv python tools/mst_once.py --config $c --warmup 0 --reps 1 > gpurun_out/p3/${c}_launches.log 2>&1; echo "launches $c rc=$?"
done
