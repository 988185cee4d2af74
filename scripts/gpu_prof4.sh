CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_polar_small" -s 1 -c 1 -o gpurun_out/prof_polar2 $CMD > gpurun_out/ncu4.log 2>&1 ; echo "ncu4 rc=$?"
