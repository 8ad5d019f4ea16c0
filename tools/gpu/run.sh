python tools/time_3xtf32.py > gpurun_out/t3x.log 2>&1; echo a=$?
