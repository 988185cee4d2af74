timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest37.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest37.log
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench37.log 2>&1; echo "bench rc=$?"
