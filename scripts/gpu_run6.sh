for cfg in 3 5 4; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg$cfg.log 2>&1; echo "cfg$cfg rc=$?"
done
