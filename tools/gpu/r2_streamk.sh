timeout 600 python -m pytest tests/test_gpu_r2.py -q -x -k "stream_k" > gpurun_out/r2_streamk_test.log 2>&1; echo "test rc=$?"
timeout 600 python tools/time_streamk.py > gpurun_out/r2_streamk_ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest20.log 2>&1; echo "suite rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench20.json 2> gpurun_out/r2_bench20.err; echo "bench rc=$?"
