timeout 900 python -m pytest tests -m gpu -q -x -k "large_rank" > gpurun_out/pytest20.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest20.log
P2G_DEBUG=1 timeout 600 python bench.py --config 3 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench20.log 2>&1; echo rc=$?
grep sweeps gpurun_out/bench20.log
ncu --set full --clock-control none --import-source on -k regex:"k_procrustes_large" -s 2 -c 1 -o gpurun_out/prof20 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu20.log 2>&1; echo "ncu rc=$?"
