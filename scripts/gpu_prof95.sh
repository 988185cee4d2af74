# final cfg2 evidence with the last accurate-path change
timeout 900 python bench.py > gpurun_out/bench95.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench95_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches95_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu95a.log 2>&1; echo "list2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mode3_sb|k_polar_small|k_mode2_sb|k_seg_spmm|k_procrustes_accurate" -s 15 -c 5 -o /tmp/prof95_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu95d.log 2>&1; echo "full2 rc=$?"
python scripts/ncu_summary.py /tmp/prof95_c2.ncu-rep > gpurun_out/full95_c2.txt 2>&1
for k in k_polar_small k_mode3_sb k_mode2_sb k_procrustes_accurate; do echo "## $k" >> gpurun_out/full95_c2_lines.txt; python scripts/ncu_lines.py /tmp/prof95_c2.ncu-rep $k 12 >> gpurun_out/full95_c2_lines.txt 2>&1; done
ncu -i /tmp/prof95_c2.ncu-rep --page raw --csv 2>/dev/null > /tmp/prof95_c2.csv
python - <<'PY' > gpurun_out/traffic95.json
import csv, json
rows = list(csv.reader(open("/tmp/prof95_c2.csv"))); h = rows[0]; u = rows[1]
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
print(json.dumps({"cfg2": d}, indent=1))
PY
