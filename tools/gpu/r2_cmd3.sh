set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest3.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err
AOL_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-peak > gpurun_out/r2_n2_matmul.json 2> gpurun_out/r2_n2_matmul.err
AOL_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --workload cg > gpurun_out/r2_n2_cg.json 2> gpurun_out/r2_n2_cg.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err
