for cfg in 3 5; do
  timeout 900 python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench17_cfg$cfg.log 2>&1; echo "cfg$cfg rc=$?"
done
