nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest60.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest60.log
timeout 600 python bench.py > gpurun_out/bench60.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench60_ref.log 2>&1; echo "ref rc=$?"
for c in 3 4 5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench60_c$c.log 2>&1; echo "bench$c rc=$?"; done
