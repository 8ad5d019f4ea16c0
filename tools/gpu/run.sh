timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tile_sum or random" > gpurun_out/t.log 2>&1; echo t=$?
timeout 300 python tools/gpu/tsum_wrap.py > gpurun_out/tw.log 2>&1
AOL_FILTER_WIDE=1 timeout 300 python tools/gpu/tsum_wrap.py >> gpurun_out/tw.log 2>&1
