P2G_DEBUG=1 CFG=4 K=200000 ITERS=6 timeout 300 python scripts/prof_large.py > gpurun_out/dbg61_c4.log 2>&1; echo "c4 rc=$?"
P2G_DEBUG=1 CFG=5 K=200000 ITERS=6 timeout 300 python scripts/prof_large.py > gpurun_out/dbg61_c5.log 2>&1; echo "c5 rc=$?"
