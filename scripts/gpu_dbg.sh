P2G_DEBUG=1 timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_dbg.log 2> gpurun_out/bench_dbg.err; echo "rc=$?"
