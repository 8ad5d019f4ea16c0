timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tile_sum" > gpurun_out/t.log 2>&1; echo t=$?
timeout 300 python tools/time_tile_sum.py > gpurun_out/tsum.log 2>&1; echo a=$?
AOL_TILE_SUM_CPASYNC=1 timeout 300 python tools/time_tile_sum.py >> gpurun_out/tsum.log 2>&1; echo a=$?
