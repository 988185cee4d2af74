timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest54.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest54.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench54.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench54_c5.log 2>&1; echo "bench5 rc=$?"
