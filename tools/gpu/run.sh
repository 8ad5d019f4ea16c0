timeout 600 python tools/time_filters.py > gpurun_out/filters.log 2>&1; echo a=$?
