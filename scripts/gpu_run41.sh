timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest41.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest41.log
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench41.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench41_c2.log 2>&1; echo "bench2 rc=$?"
