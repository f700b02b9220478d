# L2 fetch granularity / dedup threshold / offer mode experiments (device-resident, mst_once)
mkdir -p gpurun_out
python - <<'PY'
import ctypes
cu = ctypes.CDLL("libcudart.so")
v = ctypes.c_size_t()
cu.cudaFree(None)
print("default cudaLimitMaxL2FetchGranularity:", cu.cudaDeviceGetLimit(ctypes.byref(v), 5), v.value)
PY
for c in c4 c2 c3 c1 c0; do for f in 0 32 64 128; do echo -n "L2_FETCH=$f "; MST_L2_FETCH=$f timeout 300 python tools/mst_once.py --config $c --warmup 2 --reps 5 | head -1; done; done
for v in 262144 4e6 64e6; do echo -n "DEDUP_ACTIVE=$v "; MST_DEDUP_ACTIVE=$v timeout 300 python tools/mst_once.py --config c4 --warmup 2 --reps 5 | head -1; done
for v in 262144 4e6 64e6; do echo -n "DEDUP_ACTIVE=$v "; MST_DEDUP_ACTIVE=$v timeout 300 python tools/mst_once.py --config c2 --warmup 2 --reps 5 | head -1; done
echo -n "OFFER_COUNT=2 "; MST_OFFER_COUNT=2 timeout 300 python tools/mst_once.py --config c4 --warmup 2 --reps 5 | head -1
echo -n "OFFER_COUNT=0 "; MST_OFFER_COUNT=0 timeout 300 python tools/mst_once.py --config c4 --warmup 2 --reps 5 | head -1
for f in 0 32; do
MST_L2_FETCH=$f ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum --clock-control none --csv --log-file gpurun_out/c4_l2f$f.csv python tools/mst_once.py --config c4 --warmup 0 --reps 1 > /dev/null 2>&1; echo "ncu f=$f rc=$?"
done
