CFG=4 K=100000 ITERS=4 timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"k_procrustes_large_w" -s 3 -c 1 -o /tmp/prof83 python scripts/prof_large.py > gpurun_out/ncu83.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/prof83.ncu-rep > gpurun_out/full83.txt 2>&1
python scripts/ncu_lines.py /tmp/prof83.ncu-rep k_procrustes_large_w 400 > gpurun_out/lines83.txt 2>&1
ncu -i /tmp/prof83.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; r=rows[2]
for i,n in enumerate(h):
    if n in ['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__inst_executed.sum','lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum']: print(n, r[i])
" > gpurun_out/raw83.txt
