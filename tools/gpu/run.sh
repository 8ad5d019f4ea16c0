python -m pytest tests/test_gpu_parity.py -x -q -k "tile_copy" > gpurun_out/pytest_win.log 2>&1; echo pytest=$?
python bench.py --workload sweep --no-cpu > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo sweep=$?
