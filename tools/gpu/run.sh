timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_rows_shift -c 1 -o gpurun_out/rows_shift python tools/gpu/crop_probe.py > gpurun_out/ncu_rs.log 2>&1; echo a=$?
