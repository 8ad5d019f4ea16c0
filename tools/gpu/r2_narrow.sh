timeout 600 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -m gpu -q -x -k "mixed_width or stream_k or matmul" > gpurun_out/r2_narrow_tests.log 2>&1; echo "trc=$?"
for i in 1 2; do for nv in 0 1; do AOL_GEMM_NARROW=$nv timeout 300 python tools/time_streamk.py 8 2>&1 | sed "s/^/narrow=$nv /"; done; done
