python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python tools/gpu/gshift.py > gpurun_out/gshift.log 2>&1; echo a=$?
