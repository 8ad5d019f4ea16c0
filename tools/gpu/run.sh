python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py --workload cg > gpurun_out/bench_cg.json 2> gpurun_out/bench_cg.err; echo cg=$?
python bench.py --workload cg27 > gpurun_out/bench_cg27.json 2> gpurun_out/bench_cg27.err; echo cg27=$?
