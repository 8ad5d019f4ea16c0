python tools/sweep_point.py 2 dense 1e9 3 > gpurun_out/sp_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tile_copy_tma -s 1 -c 1 -o gpurun_out/prof_tma_dense python tools/sweep_point.py 2 dense 1e9 3 > gpurun_out/ncu_tma1.log 2>&1
echo a=$?
python tools/sweep_point.py 8 gaps 1e8 3 > gpurun_out/sp_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tile_copy_tma -s 1 -c 1 -o gpurun_out/prof_tma_gaps8 python tools/sweep_point.py 8 gaps 1e8 3 > gpurun_out/ncu_tma2.log 2>&1
echo b=$?
python bench.py --workload sweep --steps 20 --warmup 3 --no-points > gpurun_out/sw_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3 -c 20 --csv --log-file gpurun_out/sweep_launches.csv python bench.py --workload sweep --steps 20 --warmup 3 --no-points > gpurun_out/ncu_sw.log 2>&1
echo c=$?
