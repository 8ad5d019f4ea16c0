for sd in 501 502 503 504 505; do SEED=$sd CASES=700 timeout 900 python tools/stress_tile.py > gpurun_out/sf2_tile_$sd.log 2>&1; echo "tile $sd rc=$?"; done
for sd in 511 512 513; do SEED=$sd CASES=300 timeout 1500 python tools/stress_gemm.py > gpurun_out/sf2_gemm_$sd.log 2>&1; echo "gemm $sd rc=$?"; done
for sd in 521 522 523 524; do SEED=$sd CASES=400 timeout 900 python tools/stress_api.py > gpurun_out/sf2_api_$sd.log 2>&1; echo "api $sd rc=$?"; done
THREADS=8 CASES=200 timeout 1200 python tools/stress_threads.py > gpurun_out/sf2_thr.log 2>&1; echo "threads rc=$?"
SEED=531 CASES=600 timeout 1500 python tools/stress_sharded.py > gpurun_out/sf2_sharded.log 2>&1; echo "sharded rc=$?"
SEED=541 CASES=100 timeout 1500 python tools/stress_cg.py > gpurun_out/sf2_cg.log 2>&1; echo "cg rc=$?"
