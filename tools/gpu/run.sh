python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
python bench.py --workload downscaler > gpurun_out/bench_ds.json 2> gpurun_out/bench_ds.err; echo ds=$?
python bench.py --workload sweep > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo sweep=$?
