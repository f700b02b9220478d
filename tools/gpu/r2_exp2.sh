# c4 light-phase / beta experiments + ncu --set full of the big c4 kernels
mkdir -p gpurun_out/exp2
echo "== debug rounds default"; MST_DEBUG_ROUNDS=1 python tools/mst_once.py --config c4 --warmup 0 --reps 1 2>&1 | tail -14
echo "== debug rounds DEDUP_ACTIVE=4e6"; MST_DEDUP_ACTIVE=4e6 MST_DEBUG_ROUNDS=1 python tools/mst_once.py --config c4 --warmup 0 --reps 1 2>&1 | tail -14
for b in 0.75 1.0 1.25 1.5 2.0 3.0; do echo -n "beta=$b "; MST_FILTER_BETA=$b timeout 300 python tools/mst_once.py --config c4 --warmup 2 --reps 5 | head -1; done
MST_DEDUP_ACTIVE=4e6 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum --clock-control none --csv --log-file gpurun_out/exp2/c4_dedup4m.csv python tools/mst_once.py --config c4 --warmup 0 --reps 1 > /dev/null 2>&1; echo "ncu dedup rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application --kernel-name-base demangled \
  -k regex:"SoaView" -f -o gpurun_out/exp2/c4_soa python tools/mst_once.py --config c4 --warmup 0 --reps 1 > gpurun_out/exp2/ncu_soa.log 2>&1; echo "ncu soa rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application --kernel-name-base demangled \
  -k regex:"k_emit_staged|k_hook_decide" -f -o gpurun_out/exp2/c4_emit_hook python tools/mst_once.py --config c4 --warmup 0 --reps 1 > gpurun_out/exp2/ncu_eh.log 2>&1; echo "ncu eh rc=$?"
