set -x
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_r2.py -m gpu -x -q > gpurun_out/r2_sharded_tests.log 2>&1; echo "tests rc=$?"
i=0
for w in downscaler sweep c1 stencil; do i=$((i+1)); AOL_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700+i)) bench.py --gpus 2 --steps 5 --warmup 3 --no-peak --no-points --workload $w > gpurun_out/r2_n2_$w.json 2> gpurun_out/r2_n2_$w.err; echo "$w rc=$?"; done
