timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest7.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest7.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench7.log 2>&1; echo "bench rc=$?"
P2G_DEBUG=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench7_dbg.log 2>&1; echo "dbg rc=$?"
