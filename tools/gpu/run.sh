python -m pytest tests/test_gpu_parity.py -x -q -k "tile_copy or random_tilers or golden" > gpurun_out/pytest_b2.log 2>&1; echo pytest=$?
timeout 600 python tools/time_blocks.py > gpurun_out/blocks.log 2>&1; echo a=$?
