set -x
timeout 600 python -m pytest tests/test_gpu_r2.py -m gpu -q -x -k "more_devices" > gpurun_out/r2_dgt_test.log 2>&1; echo "dgt rc=$?"
timeout 600 python tools/time_3xtf32.py > gpurun_out/r2_3x_plain.json 2> gpurun_out/r2_3x_plain.err; echo "3x rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_3xtf32_pair -c 1 -o gpurun_out/r2_gemm_3x python tools/time_3xtf32.py > gpurun_out/r2_ncu_3x.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_gemm_3x.ncu-rep gpurun_out/r2_gemm_3x_summary.json
timeout 600 python tools/time_streamk.py 4 > gpurun_out/r2_sk4_plain.log 2>&1
AOL_GEMM_STREAMK=1 timeout 900 ncu --set full --clock-control none -k regex:k_gemm_tf32_pair -s 40 -c 1 -o gpurun_out/r2_gemm_splitk python tools/time_streamk.py 4 > gpurun_out/r2_ncu_sk.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_gemm_splitk.ncu-rep gpurun_out/r2_gemm_splitk_summary.json
