for sd in 2 3; do SEED=$sd CASES=200 timeout 900 python tools/stress_api.py > gpurun_out/sf_api_$sd.log 2>&1; echo "api seed $sd rc=$?"; done
for sd in 71 72; do SEED=$sd CASES=600 timeout 900 python tools/stress_tile.py > gpurun_out/sf_tile_$sd.log 2>&1; echo "tile seed $sd rc=$?"; done
SEED=81 CASES=250 timeout 1200 python tools/stress_gemm.py > gpurun_out/sf_gemm.log 2>&1; echo "gemm rc=$?"
SEED=91 CASES=400 timeout 900 python tools/stress_sharded.py > gpurun_out/sf_sharded.log 2>&1; echo "sharded rc=$?"
SEED=95 CASES=60 timeout 900 python tools/stress_cg.py > gpurun_out/sf_cg.log 2>&1; echo "cg rc=$?"
