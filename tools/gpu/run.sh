timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "line_tiled" > gpurun_out/t.log 2>&1; echo t=$?
