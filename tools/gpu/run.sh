python bench.py --workload c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo c1=$?
python bench.py --workload cg > gpurun_out/bench_cg.json 2> gpurun_out/bench_cg.err; echo cg=$?
python bench.py --workload cg27 > gpurun_out/bench_cg27.json 2> gpurun_out/bench_cg27.err; echo cg27=$?
