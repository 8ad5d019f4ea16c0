for u in 1 2 4; do echo U=$u; AOL_ROWS_SHIFT_U=$u timeout 300 python tools/gpu/crop_probe.py; AOL_ROWS_SHIFT_U=$u timeout 300 python tools/time_shift.py; done > gpurun_out/crop.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_plane or toroidal" > gpurun_out/t.log 2>&1; echo t=$?
