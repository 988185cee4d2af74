timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest62.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest62.log
P2G_DEBUG=1 CFG=4 K=200000 ITERS=6 timeout 300 python scripts/prof_large.py > gpurun_out/dbg62_c4.log 2>&1; echo "c4dbg rc=$?"
for c in 4 3 5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench62_c$c.log 2>&1; echo "bench$c rc=$?"; done
