set -x
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_v1.csv $CMD > gpurun_out/ncu1.log 2>&1 ; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_procrustes|k_mode2|k_nnls" -s 3 -c 3 -o gpurun_out/prof_r01_v1 $CMD > gpurun_out/ncu2.log 2>&1 ; echo "ncu2 rc=$?"
