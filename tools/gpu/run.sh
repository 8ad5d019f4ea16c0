python bench.py --workload sweep --no-points > gpurun_out/bench_sweep_e2e.json 2> gpurun_out/bench_sweep_e2e.err; echo sweep=$?
