timeout 900 python -m pytest tests -m gpu -q -x -k "large_rank" > gpurun_out/pytest22.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest22.log
P2G_DEBUG=1 python scripts/prof_large.py > gpurun_out/prof22_plain.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_procrustes_large" -s 2 -c 1 -o gpurun_out/prof22 python scripts/prof_large.py > gpurun_out/ncu22.log 2>&1; echo "ncu rc=$?"
