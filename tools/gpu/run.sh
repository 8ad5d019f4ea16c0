python -m pytest tests/test_gpu_parity.py -x -q -k "tile_copy or random or golden" > gpurun_out/pytest_sb.log 2>&1; echo pytest=$?
timeout 600 python tools/time_shift.py > gpurun_out/shift.log 2>&1; echo a=$?
