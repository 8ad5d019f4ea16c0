python -m pytest tests/test_gpu_parity.py -x -q -k "stencil" > gpurun_out/pytest_st.log 2>&1; echo pytest=$?
python tools/time_stencil_kxk.py > gpurun_out/kxk.log 2>&1; echo a=$?
