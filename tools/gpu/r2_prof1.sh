# c4 characterisation: random-access microbenchmark, per-kernel launch list with
# DRAM / L2 red+atom sectors / L1 wavefronts, --set full of the top c4 kernels
set -x
mkdir -p gpurun_out/prof1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gather_bench.cu -o tools/gather_bench && timeout 300 ./tools/gather_bench > gpurun_out/prof1/gather_bench.txt 2>&1; echo "gather rc=$?"
cat gpurun_out/prof1/gather_bench.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
for c in c4 c1; do
timeout 1200 ncu --metrics $M --clock-control none --replay-mode application --csv --log-file gpurun_out/prof1/${c}_launches.csv python tools/mst_once.py --config $c --warmup 0 --reps 1 > gpurun_out/prof1/${c}_launches.log 2>&1; echo "launches $c rc=$?"
done
timeout 2400 ncu --set full --clock-control none --import-source on --replay-mode application --kernel-name-base demangled \
  -k regex:"k_count|k_emit_staged|k_hook_decide|k_label2" -f -o gpurun_out/prof1/c4_full python tools/mst_once.py --config c4 --warmup 0 --reps 1 > gpurun_out/prof1/c4_full.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out/prof1
