timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest77.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest77.log
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench77_c5.log 2>&1; echo "bench5 rc=$?"
timeout 600 python bench.py > gpurun_out/bench77.log 2>&1; echo "bench rc=$?"
timeout 600 python scripts/first_iter.py > gpurun_out/first77.log 2>&1; echo "first rc=$?"
