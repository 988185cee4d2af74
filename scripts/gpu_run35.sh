timeout 900 python -m pytest tests -m gpu -q -x -k "large_rank" > gpurun_out/pytest35.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest35.log
P2G_DEBUG=1 python scripts/prof_large.py > gpurun_out/prof35_plain.log 2>&1; echo "plain rc=$?"
tail -4 gpurun_out/prof35_plain.log
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench35.log 2>&1; echo "bench rc=$?"
