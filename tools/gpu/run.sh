timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "tile_copy or toroidal or shift or sweep" > gpurun_out/t.log 2>&1; echo t=$?
timeout 300 python tools/time_shift.py > gpurun_out/shift.log 2>&1; echo a=$?
