P2G_DEBUG=1 CFG=4 K=200000 ITERS=6 timeout 300 python scripts/prof_large.py > gpurun_out/dbg64_c4.log 2>&1; echo "c4dbg rc=$?"
P2G_DEBUG=1 CFG=5 K=200000 ITERS=6 timeout 300 python scripts/prof_large.py > gpurun_out/dbg64_c5.log 2>&1; echo "c5dbg rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches64_c4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu64.log 2>&1; echo "ncu-list rc=$?"
