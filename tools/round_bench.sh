mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
for c in c1 c0 c2 c3 c4; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; tail -c 400 gpurun_out/bench_$c.json
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_c1_reference.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_c1_reference.json | tail -c 300
