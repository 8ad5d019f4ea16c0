timeout 300 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "3x" > gpurun_out/t_x3r.log 2>&1; echo tests=$?
for i in 1 2; do
AOL_3XTF32_FORM=wide timeout 120 python tools/time_3xtf32.py | sed 's/^/wide /'
X3_SWEEP="32:0 128:0" timeout 200 python tools/time_3xtf32.py | sed 's/^/regs /'
done
