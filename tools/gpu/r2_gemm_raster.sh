set -x
for g in 2 4 8 16 32; do AOL_GEMM_GROUP_M=$g timeout 600 python bench.py --steps 400 --warmup 10 --no-e2e --no-cpu --no-peak > gpurun_out/r2_gemm_g$g.json 2> gpurun_out/r2_gemm_g$g.err; done
AOL_GEMM_GROUP_M=8 timeout 600 python bench.py --steps 400 --warmup 10 --no-e2e --no-cpu --no-peak > gpurun_out/r2_gemm_g8b.json 2> gpurun_out/r2_gemm_g8b.err
for g in 4 8 16; do AOL_GEMM_GROUP_M=$g timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:k_gemm_tf32_pair -c 3 --csv --log-file gpurun_out/r2_gemm_ncu_g$g.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-peak --no-e2e-numpy > /dev/null 2>&1; done
