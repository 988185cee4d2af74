timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest96.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest96.log
for c in 4 3; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench96_c$c.log 2>&1; echo "bench$c rc=$?"; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench96_c5.log 2>&1; echo "bench5 rc=$?"
