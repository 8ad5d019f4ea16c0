python -m pytest tests/test_gpu_parity.py -x -q -k "streamed" > gpurun_out/pytest_str.log 2>&1; echo pytest=$?
python bench.py --workload downscaler --steps 50 --no-cpu --no-peak > gpurun_out/bench_ds.json 2> gpurun_out/bench_ds.err; echo ds=$?
