i=0
for w in matmul stencil downscaler cg; do i=$((i+1)); AOL_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29740+i)) bench.py --gpus 2 --steps 5 --warmup 3 --no-peak --no-points --no-e2e --workload $w > gpurun_out/r2_n2g_$w.json 2> gpurun_out/r2_n2g_$w.err; echo "$w rc=$?"; done
timeout 600 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x > gpurun_out/r2_fused_tests4.log 2>&1; echo "trc=$?"
