python -m pytest tests/test_gpu_parity.py -x -q -k "random_large" > gpurun_out/pytest_rl.log 2>&1; echo pytest=$?
