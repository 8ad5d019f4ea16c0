python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo s=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo t=$?
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo b=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo r=$?
timeout 900 python bench.py --workload sweep > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo w=$?
