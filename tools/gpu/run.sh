python -m pytest tests/test_gpu_parity.py -x -q -k "matmul or golden or random_tilers" > gpurun_out/pytest_ex.log 2>&1; echo pytest=$?
timeout 600 python tools/time_exact.py > gpurun_out/exact.log 2>&1; echo a=$?
