set -x
mkdir -p gpurun_out/exp22
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp22/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp22/tests.log
run() { echo -n "$* : "; env "$@" timeout 300 python tools/mst_once.py --config $C --warmup 3 --reps 20 | head -1; }
{ for C in c1 c0 c2 c4; do run MST_X=0; run MST_X=0; done; } > gpurun_out/exp22/sweep.txt 2>&1
grep -v "^+" gpurun_out/exp22/sweep.txt
for i in 1 2; do timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp22/bench_c1_$i.json 2>/dev/null; done
grep -o '"ms_per_step": [0-9.]*' gpurun_out/exp22/bench_c1_*.json
MST_TIMELINE=1 python tools/mst_once.py --config c1 --warmup 2 --reps 1 > gpurun_out/exp22/timeline_c1.txt 2>&1; grep timeline gpurun_out/exp22/timeline_c1.txt | tail -7
