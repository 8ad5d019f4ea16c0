python -m pytest tests/test_gpu_parity.py -x -q -k "tile_sum or golden or random_tilers" > gpurun_out/pytest_ts.log 2>&1; echo pytest=$?
python tools/time_tile_sum.py > gpurun_out/tsum.log 2>&1; echo a=$?
