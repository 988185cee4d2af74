timeout 600 python bench.py > gpurun_out/bench69.log 2>&1; echo "bench rc=$?"
for c in 3 4 5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench69_c$c.log 2>&1; echo "bench$c rc=$?"; done
