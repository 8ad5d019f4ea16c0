python -m pytest tests/test_gpu_parity.py -x -q -k "line_tiled or line_filter or random_tilers or fused or golden" > gpurun_out/pytest_lt.log 2>&1; echo pytest=$?
timeout 600 python tools/time_filters.py > gpurun_out/filters.log 2>&1; echo a=$?
