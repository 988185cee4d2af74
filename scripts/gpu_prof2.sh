set -x
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_polar_small|k_mode3|k_mode2|k_gram_c|k_qrows|k_nnls_thread" -s 6 -c 6 -o gpurun_out/prof_r01_v2 $CMD > gpurun_out/ncu2.log 2>&1 ; echo "ncu2 rc=$?"
