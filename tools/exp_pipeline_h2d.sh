mkdir -p gpurun_out
{
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for p in 1 0 1 0; do echo "pipeline=$p"; MST_PIPELINE_H2D=$p python tools/e2e_breakdown.py --config c1 --reps 3 --flush 2>&1 | head -3; done
python bench.py --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d['e2e'])"
} > gpurun_out/exp9.log 2>&1
