# c4/c1 launch lists with red/atom sectors, L2 hit rate, L1 wavefronts; --set full of
# the c4 offer-heavy kernels exported to CSV on the box (the .ncu-rep is too big to bring back)
set -x
mkdir -p gpurun_out/prof2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
for c in c4 c1; do
timeout 1200 ncu --metrics $M --clock-control none --replay-mode application --csv --log-file gpurun_out/prof2/${c}_launches.csv python tools/mst_once.py --config $c --warmup 0 --reps 1 > gpurun_out/prof2/${c}_launches.log 2>&1; echo "launches $c rc=$?"
done
MST_DEBUG_ROUNDS=1 python tools/mst_once.py --config c4 --warmup 1 --reps 3 > gpurun_out/prof2/c4_rounds.txt 2>&1
for a in 4e6 6.4e7; do for r in 8 2; do echo "== DEDUP_ACTIVE=$a DEDUP_MIN_RATIO=$r" >> gpurun_out/prof2/c4_dedup.txt; MST_DEDUP_ACTIVE=$a MST_DEDUP_MIN_RATIO=$r MST_DEBUG_ROUNDS=1 timeout 300 python tools/mst_once.py --config c4 --warmup 2 --reps 5 >> gpurun_out/prof2/c4_dedup.txt 2>&1; done; done
for a in 4e6 6.4e7; do echo "== c2 DEDUP_ACTIVE=$a" >> gpurun_out/prof2/c4_dedup.txt; MST_DEDUP_ACTIVE=$a timeout 300 python tools/mst_once.py --config c2 --warmup 2 --reps 5 >> gpurun_out/prof2/c4_dedup.txt 2>&1; done
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application --kernel-name-base demangled \
  -k regex:"k_emit_staged|k_count|k_hook_decide" -c 12 -f -o /tmp/c4_full python tools/mst_once.py --config c4 --warmup 0 --reps 1 > gpurun_out/prof2/c4_full.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/c4_full.ncu-rep --page raw --csv > gpurun_out/prof2/c4_full_raw.csv 2>&1
ncu -i /tmp/c4_full.ncu-rep --page details --csv > gpurun_out/prof2/c4_full_details.csv 2>&1
ls -la gpurun_out/prof2; du -sh gpurun_out
