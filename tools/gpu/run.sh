timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "random_long_rows or random_tilers" > gpurun_out/t.log 2>&1; echo t=$?
