# launch lists + ncu --set full captures, summarised on the box (reports are too big to bring back)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches71_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu71a.log 2>&1; echo "list2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches71_c4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu71b.log 2>&1; echo "list4 rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_procrustes_large_w|k_mode3_mma|k_urows|k_seg_spmm|k_nnls" -s 10 -c 5 -o /tmp/prof71_c4 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu71c.log 2>&1; echo "full4 rc=$?"
python scripts/ncu_summary.py /tmp/prof71_c4.ncu-rep > gpurun_out/full71_c4.txt 2>&1
for k in k_procrustes_large_w k_mode3_mma k_urows k_seg_spmm; do echo "## $k" >> gpurun_out/full71_c4_lines.txt; python scripts/ncu_lines.py /tmp/prof71_c4.ncu-rep $k 15 >> gpurun_out/full71_c4_lines.txt 2>&1; done
ncu -i /tmp/prof71_c4.ncu-rep --page raw --csv > /tmp/raw71.csv 2>/dev/null; python - <<'PY' > gpurun_out/raw71_c4_sel.txt
import csv
rows=list(csv.reader(open('/tmp/raw71.csv'))); h=rows[0]
want=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__inst_executed.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active','lts__t_bytes.sum','sm__warps_active.avg.pct_of_peak_sustained_active']
idx=[h.index(w) for w in want if w in h]
for r in rows[2:]:
    print(' | '.join(f'{h[i]}={r[i]}' for i in idx))
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mode3_sb|k_polar_small|k_mode2_sb|k_seg_spmm|k_procrustes_accurate" -s 15 -c 5 -o /tmp/prof71_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu71d.log 2>&1; echo "full2 rc=$?"
python scripts/ncu_summary.py /tmp/prof71_c2.ncu-rep > gpurun_out/full71_c2.txt 2>&1
du -sh gpurun_out
