timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "line" > gpurun_out/t.log 2>&1; echo t=$?
timeout 300 python tools/time_filters.py > gpurun_out/filters.log 2>&1; echo a=$?
