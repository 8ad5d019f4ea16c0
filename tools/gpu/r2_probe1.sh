set -x
timeout 600 python -m pytest tests/test_dsl_models.py tests/test_codegen_b200.py -m gpu -x -q > gpurun_out/r2_newtests.log 2>&1
P="1:gaps:1e7 1:dense:1e7 2:dense:1e7 2:overlap:1e7 2:gaps:1e7 4:gaps:1e7 8:gaps:1e7 16:gaps:1e7 16:gaps:1e8 8:gaps:1e8 16:dense:1e7 32:rowstride:1e7 4:rowstride:1e7"
timeout 300 python tools/sweep_probe.py $P > gpurun_out/probe1_default.log 2>&1
timeout 300 python tools/sweep_probe.py --gran 32 8:gaps:1e8 16:gaps:1e8 8:gaps:1e7 16:gaps:1e7 4:gaps:1e8 > gpurun_out/probe1_g32.log 2>&1
timeout 300 python tools/sweep_probe.py --gran 64 8:gaps:1e8 16:gaps:1e8 8:gaps:1e7 16:gaps:1e7 4:gaps:1e8 > gpurun_out/probe1_g64.log 2>&1
timeout 300 python tools/sweep_probe.py --gran 0 8:gaps:1e8 16:gaps:1e8 > gpurun_out/probe1_g0.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_tile_copy_tma --csv --log-file gpurun_out/probe1_ncu_g64.csv python tools/sweep_probe.py --gran 64 16:gaps:1e7 > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_tile_copy_tma --csv --log-file gpurun_out/probe1_ncu_def.csv python tools/sweep_probe.py 16:gaps:1e7 > /dev/null 2>&1
