set -x
timeout 600 python tools/sweep_dram_ncu.py run > gpurun_out/sweep_dram_plain.log 2>&1 || exit 1
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sweep_dram.csv python tools/sweep_dram_ncu.py run > gpurun_out/sweep_dram_ncu.log 2>&1
python tools/sweep_dram_ncu.py parse gpurun_out/sweep_dram.csv > gpurun_out/r2_sweep_dram.json 2> gpurun_out/sweep_dram_parse.err
cp gpurun_out/r2_sweep_dram.json profiles/r2_sweep_dram.json
timeout 900 python bench.py --workload sweep --steps 20 --warmup 5 --no-e2e > gpurun_out/r2_bench_sweep2.json 2> gpurun_out/r2_bench_sweep2.err
