for sd in 31 32 33 34 35 36 37 38; do SEED=$sd CASES=600 timeout 900 python tools/stress_tile.py > gpurun_out/st_tile_$sd.log 2>&1; echo "tile seed $sd rc=$?"; done
for sd in 41 42 43; do SEED=$sd CASES=250 timeout 1200 python tools/stress_gemm.py > gpurun_out/st_gemm_$sd.log 2>&1; echo "gemm seed $sd rc=$?"; done
SEED=51 CASES=500 timeout 900 python tools/stress_sharded.py > gpurun_out/st_sharded.log 2>&1; echo "sharded rc=$?"
SEED=61 CASES=80 timeout 900 python tools/stress_cg.py > gpurun_out/st_cg.log 2>&1; echo "cg rc=$?"
