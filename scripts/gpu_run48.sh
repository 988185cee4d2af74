timeout 900 python -m pytest tests -m gpu -q -k "large_rank or deterministic" > gpurun_out/pytest48.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest48.log
P2G_DEBUG=1 timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench48.log 2>&1; echo "bench rc=$?"
grep sweeps gpurun_out/bench48.log | tail -2
