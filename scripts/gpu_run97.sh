timeout 600 python -m pytest tests -m gpu -q -x -k "large_rank or cfg5 or bitwise or state" > gpurun_out/pytest97.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest97.log
for c in 4 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench97_c$c.log 2>&1; echo "bench$c rc=$?"; done
