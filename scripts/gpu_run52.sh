timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest52.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest52.log
P2G_DEBUG=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench52d.log 2>&1; grep sweeps gpurun_out/bench52d.log | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench52.log 2>&1; echo "bench rc=$?"
