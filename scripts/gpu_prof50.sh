timeout 900 python bench.py > gpurun_out/bench_full_r01b.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_r01b.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu30a.log 2>&1; echo "ncu-list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_mode3_sb|k_polar_small|k_mode2_sb|k_seg_spmm|k_procrustes_accurate" -s 15 -c 5 -o gpurun_out/prof_r01b_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu30b.log 2>&1; echo "ncu-full rc=$?"
for cfg in 3 5 4; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg${cfg}_r01b.log 2>&1; echo "cfg$cfg rc=$?"
done
