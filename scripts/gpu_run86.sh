timeout 600 python -m pytest tests -m gpu -q -x -k "large_rank or bitwise or cfg5" > gpurun_out/pytest86.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest86.log
for c in 4 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench86_c$c.log 2>&1; echo "bench$c rc=$?"; done
