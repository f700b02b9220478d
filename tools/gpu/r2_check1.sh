set -x
nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c4" > gpurun_out/t1.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/t1.log
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err; echo "c1 rc=$?"
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --impl reference --config c4 --steps 3 --warmup 1 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err; echo "ref rc=$?"
