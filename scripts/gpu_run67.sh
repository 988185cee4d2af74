timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest67.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest67.log
for c in 4 3; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench67_c$c.log 2>&1; echo "bench$c rc=$?"; done
