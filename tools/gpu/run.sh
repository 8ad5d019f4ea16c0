for p in "0 0" "1 0" "0 1" "1 2" "3 3"; do timeout 60 python tools/gpu/plane_probe.py $p 2>&1 | tail -2; done > gpurun_out/probe.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_plane or toroidal or block_tilers or tile_copy" > gpurun_out/t.log 2>&1; echo t=$?
timeout 300 python tools/time_shift.py > gpurun_out/shift.log 2>&1; echo a=$?
AOL_COPY_NO_PLANE=1 timeout 300 python tools/time_shift.py >> gpurun_out/shift.log 2>&1; echo b=$?
