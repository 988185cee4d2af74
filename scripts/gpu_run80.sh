timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest80.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest80.log
timeout 900 python bench.py > gpurun_out/bench80.log 2>&1; echo "bench rc=$?"
for c in 3 4 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench80_c$c.log 2>&1; echo "bench$c rc=$?"; done
P2G_TIMING=1 timeout 600 python scripts/e2e_timing.py > gpurun_out/e2e80.log 2>&1; echo "e2e rc=$?"
