CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:"k_mode2_sb|k_mode3_sb|k_polar_small|k_procrustes_accurate" -s 8 -c 4 -o gpurun_out/prof8 $CMD > gpurun_out/ncu8.log 2>&1; echo "ncu rc=$?"
