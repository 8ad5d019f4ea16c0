i=0
for w in matmul stencil; do i=$((i+1)); AOL_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29800+i)) bench.py --impl reference --gpus 2 --steps 2 --warmup 1 --workload $w > gpurun_out/n2r_$w.json 2> gpurun_out/n2r_$w.err; echo "$w rc=$?"; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/n1r_matmul.json 2>/dev/null; echo "n1 rc=$?"
