CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/prof5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu5a.log 2>&1; echo "ncu5a rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_polar_small|k_mode2_qf|k_mode3_qf|k_nnls_thread|k_procrustes_accurate" -s 5 -c 5 -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu5b.log 2>&1; echo "ncu5b rc=$?"
