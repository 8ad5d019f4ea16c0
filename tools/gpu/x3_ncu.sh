ncu --set full --clock-control none --import-source on -k regex:k_gemm_3xtf32_pair -c 1 -o gpurun_out/x3_tmemA python tools/time_3xtf32.py > gpurun_out/x3_ncu.log 2>&1
echo ncu=$?
