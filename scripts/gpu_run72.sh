timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest72.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest72.log
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench72_c4.log 2>&1; echo "bench4 rc=$?"
timeout 600 python bench.py > gpurun_out/bench72.log 2>&1; echo "bench rc=$?"
