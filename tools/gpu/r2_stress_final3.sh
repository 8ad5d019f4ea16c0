for sd in 601 602 603 604 605; do SEED=$sd CASES=700 timeout 900 python tools/stress_tile.py > gpurun_out/sf3_tile_$sd.log 2>&1; echo "tile $sd rc=$?"; done
for sd in 611 612 613; do SEED=$sd CASES=300 timeout 1500 python tools/stress_gemm.py > gpurun_out/sf3_gemm_$sd.log 2>&1; echo "gemm $sd rc=$?"; done
for sd in 621 622 623 624; do SEED=$sd CASES=400 timeout 900 python tools/stress_api.py > gpurun_out/sf3_api_$sd.log 2>&1; echo "api $sd rc=$?"; done
THREADS=8 CASES=200 timeout 1200 python tools/stress_threads.py > gpurun_out/sf3_thr.log 2>&1; echo "threads rc=$?"
SEED=631 CASES=600 timeout 1500 python tools/stress_sharded.py > gpurun_out/sf3_sharded.log 2>&1; echo "sharded rc=$?"
SEED=641 CASES=100 timeout 1500 python tools/stress_cg.py > gpurun_out/sf3_cg.log 2>&1; echo "cg rc=$?"
