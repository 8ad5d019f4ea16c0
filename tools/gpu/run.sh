python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-peak > gpurun_out/gemm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 1 -o gpurun_out/prof_gemm_epi python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-peak > gpurun_out/ncu_gemm.log 2>&1
echo ncu=$?
python bench.py --steps 20 --warmup 3 --no-cpu --no-peak > gpurun_out/mm_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/matmul_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-peak > gpurun_out/ncu_mm2.log 2>&1
echo launches=$?
AOL_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu --no-peak > gpurun_out/n2.json 2> gpurun_out/n2.err
echo n2=$?
