mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c1 c0 c2 c3 c4; do python tools/mst_once.py --config $c --warmup 3 --reps 10 | head -1; done
for f in write write+read write write+read; do python bench.py --flush $f --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['frac'])"; done
} > gpurun_out/exp6.log 2>&1
