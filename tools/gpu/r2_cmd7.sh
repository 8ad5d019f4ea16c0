set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest7.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke7.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench7.json 2> gpurun_out/r2_bench7.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref7.json 2> gpurun_out/r2_ref7.err
for w in stencil downscaler sweep cg c1; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r2_bench7_$w.json 2> gpurun_out/r2_bench7_$w.err; done
AOL_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-peak > gpurun_out/r2_n2_matmul7.json 2> gpurun_out/r2_n2_matmul7.err
