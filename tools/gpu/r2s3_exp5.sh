# filter beta sweep
mkdir -p gpurun_out/s3e5
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 2 --reps 5 | head -1; }
{ for C in c4 c3 c2; do for b in 1 1.5 2 2.5 3 4; do run MST_FILTER_BETA=$b; done; done; } > gpurun_out/s3e5/sweep.txt 2>&1
cat gpurun_out/s3e5/sweep.txt
