#!/bin/bash
# One GPU evidence pass: GPU suite, default bench, reference arm, ncu launch list.
# Usage (from the repo root, under gpurun): bash scripts/gpu_round.sh TAG [tests|bench|ref|launches]...
set -u
TAG=${1:-r02}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
for step in "$@"; do
  case $step in
    tests) timeout 3000 python -m pytest tests -m gpu -q -x --durations=25 > $OUT/gputest.log 2>&1; echo "tests rc=$?" ;;
    bench) timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" ;;
    ref) timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?" ;;
    launches) timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
        > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?" ;;
  esac
done
