for sd in 201 202; do SEED=$sd CASES=700 timeout 900 python tools/stress_tile.py > gpurun_out/sz_tile_$sd.log 2>&1; echo "tile $sd rc=$?"; done
for sd in 211 212; do SEED=$sd CASES=250 timeout 1200 python tools/stress_gemm.py > gpurun_out/sz_gemm_$sd.log 2>&1; echo "gemm $sd rc=$?"; done
for sd in 221 222 223; do SEED=$sd CASES=300 timeout 900 python tools/stress_api.py > gpurun_out/sz_api_$sd.log 2>&1; echo "api $sd rc=$?"; done
THREADS=6 CASES=150 timeout 900 python tools/stress_threads.py > gpurun_out/sz_thr.log 2>&1; echo "threads rc=$?"
SEED=231 CASES=400 timeout 1200 python tools/stress_sharded.py > gpurun_out/sz_sharded.log 2>&1; echo "sharded rc=$?"
SEED=241 CASES=60 timeout 1200 python tools/stress_cg.py > gpurun_out/sz_cg.log 2>&1; echo "cg rc=$?"
