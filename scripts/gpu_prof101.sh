# final round-1 evidence
timeout 900 python bench.py > gpurun_out/bench101.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench101_ref.log 2>&1; echo "ref rc=$?"
for c in 3 4 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench101_c$c.log 2>&1; echo "bench$c rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches101_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu101a.log 2>&1; echo "list2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches101_c4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu101b.log 2>&1; echo "list4 rc=$?"
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_mode3_sb|k_polar_small|k_mode2_sb|k_seg_spmm|k_procrustes_accurate" -s 15 -c 5 -o /tmp/prof101_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu101d.log 2>&1; echo "full2 rc=$?"
python scripts/ncu_summary.py /tmp/prof101_c2.ncu-rep > gpurun_out/full101_c2.txt 2>&1
for k in k_polar_small k_mode3_sb k_mode2_sb k_procrustes_accurate; do echo "## $k" >> gpurun_out/full101_c2_lines.txt; python scripts/ncu_lines.py /tmp/prof101_c2.ncu-rep $k 12 >> gpurun_out/full101_c2_lines.txt 2>&1; done
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:"k_procrustes_large_w|k_mode3_mma|k_urows|k_seg_spmm|k_nnls" -s 10 -c 5 -o /tmp/prof101_c4 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu101c.log 2>&1; echo "full4 rc=$?"
python scripts/ncu_summary.py /tmp/prof101_c4.ncu-rep > gpurun_out/full101_c4.txt 2>&1
for k in k_procrustes_large_w k_mode3_mma k_seg_spmm; do echo "## $k" >> gpurun_out/full101_c4_lines.txt; python scripts/ncu_lines.py /tmp/prof101_c4.ncu-rep $k 15 >> gpurun_out/full101_c4_lines.txt 2>&1; done
for rep in /tmp/prof101_c2 /tmp/prof101_c4; do ncu -i $rep.ncu-rep --page raw --csv 2>/dev/null > $rep.csv; done
python - <<'PY' > gpurun_out/raw101_sel.txt
import csv
for rep in ("/tmp/prof101_c2.csv", "/tmp/prof101_c4.csv"):
    rows=list(csv.reader(open(rep))); h=rows[0]; u=rows[1]
    want=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__inst_executed.sum','sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active']
    idx=[h.index(w) for w in want if w in h]
    for r in rows[2:]:
        print(' | '.join(f'{h[i]}={r[i]}{u[i] if u[i] not in ("", "inst") else ""}' for i in idx)[:900])
PY
python - <<'PY' > gpurun_out/traffic101.json
import csv, json
out = {}
for cfg, rep in (("cfg2", "/tmp/prof101_c2.csv"), ("cfg4", "/tmp/prof101_c4.csv")):
    rows = list(csv.reader(open(rep))); h = rows[0]; u = rows[1]
    ki, rd, wr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    d = {}
    for r in rows[2:]:
        try:
            b = float(r[rd]) * scale.get(u[rd], 1) + float(r[wr]) * scale.get(u[wr], 1)
        except ValueError:
            continue
        name = r[ki].split("(")[0].split("::")[-1].split("<")[0]
        d[name] = d.get(name, 0.0) + b
    out[cfg] = d
print(json.dumps(out, indent=1))
PY
