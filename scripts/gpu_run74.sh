timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest74.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest74.log
P2G_TIMING=1 timeout 600 python scripts/e2e_timing.py > gpurun_out/e2e74.log 2>&1; echo "e2e rc=$?"
timeout 600 python bench.py > gpurun_out/bench74.log 2>&1; echo "bench rc=$?"
