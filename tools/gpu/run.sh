timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "tile_copy or sweep or rowstride" > gpurun_out/t.log 2>&1; echo t=$?
timeout 900 python bench.py --workload sweep > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo s=$?
