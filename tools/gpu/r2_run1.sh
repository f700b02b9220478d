# round 2 re-entry: full -m gpu suite (c4 golden included), smoke, c4 + c1 bench, reference arm
set -x
mkdir -p gpurun_out
nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/t1.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/t1.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err; echo "c1 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err; echo "ref rc=$?"
cat gpurun_out/b_c4.json gpurun_out/b_c1.json gpurun_out/ref_c4.json | cut -c1-600
