timeout 900 python bench.py > gpurun_out/bench102.log 2>&1; echo "bench rc=$?"
for c in 3 4 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench102_c$c.log 2>&1; echo "bench$c rc=$?"; done
