timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest18.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest18.log
for cfg in 3 5; do
  timeout 900 python bench.py --config $cfg --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench18_cfg$cfg.log 2>&1; echo "cfg$cfg rc=$?"
done
