timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest90.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest90.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench90.log 2>&1; echo "bench rc=$?"
