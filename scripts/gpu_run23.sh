timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest23.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest23.log
P2G_DEBUG=1 timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench23.log 2>&1; echo rc=$?
grep sweeps gpurun_out/bench23.log | tail -3
