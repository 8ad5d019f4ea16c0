python -m pytest tests/test_gpu_parity.py -x -q -k "float64_tile_ops or index_and_value or dtype_variants or dot_reuse" > gpurun_out/pytest_new.log 2>&1; echo pytest=$?
