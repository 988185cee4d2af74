ncu --set full --clock-control none --import-source on -k regex:"k_mode3" -s 1 -c 1 -o gpurun_out/prof39 python scripts/prof_large.py > gpurun_out/ncu39.log 2>&1; echo "ncu rc=$?"
