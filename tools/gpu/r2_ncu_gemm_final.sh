set -x
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-peak > gpurun_out/r2_ncu_plain.json 2>gpurun_out/r2_ncu_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_matmul_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-peak > gpurun_out/r2_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tf32_pair -s 3 -c 1 -o gpurun_out/r2_gemm_pair python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-peak > gpurun_out/r2_ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_gemm_pair.ncu-rep gpurun_out/r2_gemm_pair_summary.json
