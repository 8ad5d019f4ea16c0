set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_full_gputest.log 2>&1; echo "suite rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_full_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_full_bench.json 2> gpurun_out/r2_full_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_full_ref.json 2> gpurun_out/r2_full_ref.err; echo "ref rc=$?"
for w in stencil downscaler sweep cg cg27 c1; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r2_full_bench_$w.json 2> gpurun_out/r2_full_bench_$w.err; echo "$w rc=$?"; done
for w in stencil downscaler sweep cg; do timeout 600 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > gpurun_out/r2_full_ref_$w.json 2> gpurun_out/r2_full_ref_$w.err; done
timeout 900 python bench.py --steps 400 --warmup 10 --no-e2e --no-e2e-numpy > gpurun_out/r2_full_bench_400.json 2> gpurun_out/r2_full_bench_400.err; echo "400 rc=$?"
