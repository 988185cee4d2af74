P2G_DEBUG=1 python scripts/prof_large.py > gpurun_out/prof34_plain.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_procrustes_large" -s 2 -c 1 -o gpurun_out/prof34 python scripts/prof_large.py > gpurun_out/ncu34.log 2>&1; echo "ncu rc=$?"
