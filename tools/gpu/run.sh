timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hline_stream -c 1 -o gpurun_out/line_stream python tools/time_filters.py > gpurun_out/ncu_ls.log 2>&1; echo a=$?
