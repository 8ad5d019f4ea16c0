SEED=12 CASES=200 timeout 1200 python tools/stress_gemm.py > gpurun_out/stress_gemm_x3r.log 2>&1; echo stress=$?
timeout 200 python tools/diag_3x_wide.py > gpurun_out/diag_x3r.log 2>&1; echo diag=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_3xtf32_regs -c 1 -o gpurun_out/x3_regs python tools/time_3xtf32.py > gpurun_out/x3r_ncu.log 2>&1; echo ncu=$?
