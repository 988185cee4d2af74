timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest85.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest85.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke85.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke85.log
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench85_c4.log 2>&1; echo "bench4 rc=$?"
