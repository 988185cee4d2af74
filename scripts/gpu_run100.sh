timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest100.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest100.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench100.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench100_c5.log 2>&1; echo "bench5 rc=$?"
