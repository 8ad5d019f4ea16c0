timeout 300 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "3x" > gpurun_out/t_x3w.log 2>&1; echo tests=$?
timeout 200 python tools/diag_3x_wide.py 2>&1 | grep "bits"
for i in 1 2; do
AOL_3XTF32_WIDE=0 timeout 120 python tools/time_3xtf32.py | sed 's/^/narrow /'
X3_SWEEP="32:0 128:0" timeout 200 python tools/time_3xtf32.py | sed 's/^/wide /'
done
