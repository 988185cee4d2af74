timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest78.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest78.log
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench78_c4.log 2>&1; echo "bench4 rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench78.log 2>&1; echo "bench rc=$?"
