CFG=4 K=60000 ITERS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_procrustes_large_w" -s 2 -c 1 -o gpurun_out/prof63_large python scripts/prof_large.py > gpurun_out/ncu63.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu63.log
