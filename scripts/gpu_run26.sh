timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest26.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest26.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench26.log 2>&1; echo "bench rc=$?"
