set -x
mkdir -p gpurun_out/exp14
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 2 --reps 5 | head -1; }
{ for C in c4; do run MST_L2_PERSIST_MB=0; for v in 32 64 96; do run MST_L2_PERSIST_MB=$v; done; run MST_L2_PERSIST_MB=0; done; } > gpurun_out/exp14/sweep.txt 2>&1
grep -v "^+" gpurun_out/exp14/sweep.txt
python -c "
import ctypes; cu=ctypes.CDLL('libcudart.so'); v=ctypes.c_int()
cu.cudaDeviceGetAttribute(ctypes.byref(v), 79, 0); print('maxPersistingL2', v.value)
cu.cudaDeviceGetAttribute(ctypes.byref(v), 80, 0); print('maxAccessPolicyWindow', v.value)"
