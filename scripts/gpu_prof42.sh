ncu --set full --clock-control none --import-source on -k regex:"k_procrustes_large_w" -s 2 -c 1 -o gpurun_out/prof49 python scripts/prof_large.py > gpurun_out/ncu42.log 2>&1; echo "ncu rc=$?"
