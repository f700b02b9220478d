set -x
mkdir -p gpurun_out/s3e1
timeout 300 ./tools/dsmem_bench > gpurun_out/s3e1/dsmem.txt 2>&1
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 3 --reps 10 | head -1; }
{ for C in c4 c2; do run MST_DEDUP_ACTIVE=262144; run MST_DEDUP_ACTIVE=8000000; run MST_DEDUP_ACTIVE=8000000 MST_DEDUP_CAP_LOG2=23; done; } > gpurun_out/s3e1/sweep.txt 2>&1
