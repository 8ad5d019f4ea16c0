python -m pytest tests/test_gpu_parity.py -x -q -k "tile_copy" > gpurun_out/pytest_s2.log 2>&1; echo pytest=$?
python tools/sweep_time.py "1:gaps:100000000" "1:gaps:1000000000" "2:gaps:100000000" > gpurun_out/s2.log 2>&1; echo t=$?
