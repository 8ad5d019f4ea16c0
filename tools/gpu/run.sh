python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
