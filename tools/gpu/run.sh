python -m pytest tests/test_gpu_parity.py -x -q -k "box_pool or stencil or random_tilers" > gpurun_out/pytest_bp.log 2>&1; echo pytest=$?
timeout 600 python tools/time_filters.py > gpurun_out/filters.log 2>&1; echo a=$?
