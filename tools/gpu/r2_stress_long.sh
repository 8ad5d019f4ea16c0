for sd in 101 102 103 104; do SEED=$sd CASES=300 timeout 1500 python tools/stress_gemm.py > gpurun_out/sl_gemm_$sd.log 2>&1; echo "gemm $sd rc=$?"; done
for sd in 111 112 113; do SEED=$sd CASES=250 timeout 900 python tools/stress_api.py > gpurun_out/sl_api_$sd.log 2>&1; echo "api $sd rc=$?"; done
for sd in 121 122 123 124; do SEED=$sd CASES=700 timeout 900 python tools/stress_tile.py > gpurun_out/sl_tile_$sd.log 2>&1; echo "tile $sd rc=$?"; done
SEED=131 CASES=500 timeout 1200 python tools/stress_sharded.py > gpurun_out/sl_sharded.log 2>&1; echo "sharded rc=$?"
SEED=141 CASES=100 timeout 1200 python tools/stress_cg.py > gpurun_out/sl_cg.log 2>&1; echo "cg rc=$?"
