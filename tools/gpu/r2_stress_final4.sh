for sd in 801 802 803 804 805; do SEED=$sd CASES=700 timeout 900 python tools/stress_tile.py > gpurun_out/sf4_tile_$sd.log 2>&1; echo "tile $sd rc=$?"; done
for sd in 811 812 813; do SEED=$sd CASES=300 timeout 1500 python tools/stress_gemm.py > gpurun_out/sf4_gemm_$sd.log 2>&1; echo "gemm $sd rc=$?"; done
for sd in 821 822 823 824; do SEED=$sd CASES=400 timeout 900 python tools/stress_api.py > gpurun_out/sf4_api_$sd.log 2>&1; echo "api $sd rc=$?"; done
THREADS=8 CASES=200 timeout 1200 python tools/stress_threads.py > gpurun_out/sf4_thr.log 2>&1; echo "threads rc=$?"
SEED=831 CASES=600 timeout 1500 python tools/stress_sharded.py > gpurun_out/sf4_sharded.log 2>&1; echo "sharded rc=$?"
SEED=841 CASES=100 timeout 1500 python tools/stress_cg.py > gpurun_out/sf4_cg.log 2>&1; echo "cg rc=$?"
