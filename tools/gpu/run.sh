python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "matmul or c2" > gpurun_out/pytest_mm.log 2>&1; echo pytest=$?
for e in 0 1 0 1; do
AOL_GEMM_EPI_SMEM=$e python bench.py --steps 2000 --warmup 20 --no-e2e --no-cpu --no-peak > gpurun_out/mm_epi$e.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/mm_epi$e.json')); print('epi=$e', round(d['value'],1), d['clocks'])" >> gpurun_out/mm_ab.log
done
