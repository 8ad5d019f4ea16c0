python -m pytest tests/test_gpu_parity.py -x -q -k "tile_copy" > gpurun_out/pytest_tp.log 2>&1; echo pytest=$?
