set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest6.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench6.json 2> gpurun_out/r2_bench6.err
