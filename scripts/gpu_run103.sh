timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest103.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest103.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke103.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke103.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench103.log 2>&1; echo "bench rc=$?"
