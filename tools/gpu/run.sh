timeout 600 python tools/time_batched.py > gpurun_out/batched.log 2>&1; echo a=$?
