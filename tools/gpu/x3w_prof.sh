timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_x3w.json 2> gpurun_out/bench_x3w.err; echo bench=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_3xtf32_wide -c 1 -o gpurun_out/x3_wide python tools/time_3xtf32.py > gpurun_out/x3w_ncu.log 2>&1; echo ncu=$?
