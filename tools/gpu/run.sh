python -m pytest tests/test_gpu_parity.py -x -q -k "tile_copy" > gpurun_out/pytest_tp.log 2>&1; echo pytest=$?
for m in 8 16 32 64; do python tools/sweep_point.py $m rowstride 1e8 3 >> gpurun_out/sp_tp.log 2>&1; done
python bench.py --workload sweep --no-cpu > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo sweep=$?
