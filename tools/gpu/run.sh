for w in matmul downscaler cg sweep; do
AOL_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 2 --workload $w --steps 10 --warmup 3 --no-cpu --no-peak --no-points > gpurun_out/n2_$w.json 2> gpurun_out/n2_$w.err
echo $w=$?
done
