timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_sum_cols -c 1 -o gpurun_out/tsum_cols python tools/time_tile_sum.py > gpurun_out/ncu_ts.log 2>&1; echo b=$?
