timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x > gpurun_out/r2_fused_tests.log 2>&1; echo "trc=$?"
i=0
for w in matmul stencil downscaler; do i=$((i+1)); AOL_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29730+i)) bench.py --gpus 2 --steps 5 --warmup 3 --no-peak --no-points --workload $w > gpurun_out/r2_n2f_$w.json 2> gpurun_out/r2_n2f_$w.err; echo "$w rc=$?"; done
