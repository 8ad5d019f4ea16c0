python tools/prof_c1.py > gpurun_out/prof_c1.log 2>&1; echo a=$?
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
