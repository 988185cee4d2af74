timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches88_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu88a.log 2>&1; echo "list2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mode2_sb|k_mode3_sb" -s 6 -c 2 -o /tmp/prof88 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu88b.log 2>&1; echo "full rc=$?"
python scripts/ncu_summary.py /tmp/prof88.ncu-rep > gpurun_out/full88.txt 2>&1
for k in k_mode2_sb k_mode3_sb; do echo "## $k" >> gpurun_out/lines88.txt; python scripts/ncu_lines.py /tmp/prof88.ncu-rep $k 14 >> gpurun_out/lines88.txt 2>&1; done
