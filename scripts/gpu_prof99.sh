# R=40 evidence after the diagonal-block change
for c in 3 4 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench99_c$c.log 2>&1; echo "bench$c rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches99_c4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu99b.log 2>&1; echo "list4 rc=$?"
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:"k_procrustes_large_w|k_mode3_mma|k_urows|k_seg_spmm|k_nnls" -s 10 -c 5 -o /tmp/prof99_c4 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu99c.log 2>&1; echo "full4 rc=$?"
python scripts/ncu_summary.py /tmp/prof99_c4.ncu-rep > gpurun_out/full99_c4.txt 2>&1
for k in k_procrustes_large_w k_mode3_mma k_seg_spmm; do echo "## $k" >> gpurun_out/full99_c4_lines.txt; python scripts/ncu_lines.py /tmp/prof99_c4.ncu-rep $k 15 >> gpurun_out/full99_c4_lines.txt 2>&1; done
ncu -i /tmp/prof99_c4.ncu-rep --page raw --csv 2>/dev/null > /tmp/prof99_c4.csv
python - <<'PY' > gpurun_out/raw99_sel.txt
import csv
rows=list(csv.reader(open("/tmp/prof99_c4.csv"))); h=rows[0]; u=rows[1]
want=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__inst_executed.sum','sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active']
idx=[h.index(w) for w in want if w in h]
for r in rows[2:]:
    print(' | '.join(f'{h[i]}={r[i]}{u[i] if u[i] not in ("", "inst") else ""}' for i in idx)[:900])
PY
