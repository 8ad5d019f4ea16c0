timeout 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -m gpu -q -x -k "gemm2d or streamed" > gpurun_out/r2_gemm2d_tests.log 2>&1; echo "trc=$?"
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-peak --e2e-steps 20 > gpurun_out/r2_gemm2d_bench_$i.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r2_gemm2d_bench_$i.json').read().splitlines()[0]); print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],2), 'e2e_numpy', round(d['e2e_numpy']['value'],1))"; done
