timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest28.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest28.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench28.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench28_c3.log 2>&1; echo "bench3 rc=$?"
