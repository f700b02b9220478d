# pipelined single-pass split / heavy filter A/B
mkdir -p gpurun_out/s3e3
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 3 --reps 10 | head -1; }
{ for C in c4 c3 c2; do run MST_SPLIT1=0; run MST_SPLIT1=1 MST_LAZY_ENDS=0; run MST_SPLIT1=1; done; } > gpurun_out/s3e3/sweep.txt 2>&1
cat gpurun_out/s3e3/sweep.txt
MST_TIMELINE=1 timeout 300 python tools/mst_once.py --config c4 --warmup 1 --reps 1 > gpurun_out/s3e3/timeline_c4.txt 2>&1
