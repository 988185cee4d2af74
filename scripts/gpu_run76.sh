P2G_DEBUG=1 CFG=5 K=200000 ITERS=5 timeout 300 python scripts/prof_large.py > gpurun_out/dbg76_c5.log 2>&1; echo "c5 rc=$?"
CFG=5 K=200000 ITERS=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_procrustes_accurate" -s 3 -c 1 -o /tmp/prof76 python scripts/prof_large.py > gpurun_out/ncu76.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/prof76.ncu-rep > gpurun_out/full76.txt 2>&1
python scripts/ncu_lines.py /tmp/prof76.ncu-rep k_procrustes_accurate 30 > gpurun_out/lines76.txt 2>&1
