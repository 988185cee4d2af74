timeout 600 python -m pytest tests -m gpu -q -x -k "large_rank or bitwise or cfg5" > gpurun_out/pytest65.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest65.log
CFG=4 K=200000 ITERS=6 timeout 300 python scripts/prof_large.py > gpurun_out/dbg65_c4.log 2>&1; echo "c4 rc=$?"
CFG=5 K=200000 ITERS=6 timeout 300 python scripts/prof_large.py > gpurun_out/dbg65_c5.log 2>&1; echo "c5 rc=$?"
