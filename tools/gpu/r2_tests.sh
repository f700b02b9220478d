# full -m gpu suite + smoke on one B200
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/t2.log 2>&1; echo "tests rc=$?"
tail -8 gpurun_out/t2.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?"
