timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest91.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest91.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench91.log 2>&1; echo "bench rc=$?"
timeout 600 python scripts/first_iter.py > gpurun_out/first91.log 2>&1; echo "first rc=$?"
