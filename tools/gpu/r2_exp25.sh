set -x
mkdir -p gpurun_out/exp25
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp25/tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/exp25/tests.log
