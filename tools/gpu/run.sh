timeout 300 python tools/gpu/crop_probe.py > gpurun_out/crop.log 2>&1; echo a=$?
timeout 300 python tools/time_shift.py >> gpurun_out/crop.log 2>&1; echo b=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_plane or toroidal" > gpurun_out/t.log 2>&1; echo t=$?
