#!/bin/bash
# ncu --set full captures of the cfg4 (or CFG/K) loop kernels, one launch each, plus the
# sweep histograms of a P2G_DEBUG run.  Usage (under gpurun): bash scripts/gpu_ncu.sh TAG [K] [kernels...]
set -u
TAG=${1:-ncu_r02}; K=${2:-1000000}; shift; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
export CFG=${CFG:-4} RANK=${RANK:-40} K ITERS=${ITERS:-5}
P2G_DEBUG=1 P2G_TIMING=1 timeout 900 python scripts/prof_large.py > $OUT/debug_run.log 2>&1; echo "debug rc=$?"
for kern in "$@"; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$kern --launch-skip ${SKIP:-3} --launch-count 1 \
    -f -o $OUT/$kern python scripts/prof_large.py > $OUT/$kern.log 2>&1; echo "$kern rc=$?"
done
ls -la $OUT
