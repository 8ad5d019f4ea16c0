timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo t=$?
timeout 900 python bench.py --workload sweep > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo s=$?
