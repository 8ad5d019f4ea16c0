python -m pytest tests/test_gpu_parity.py -x -q -k "cg or spmv or identity or dot or loop or scalar" > gpurun_out/pytest_cg.log 2>&1; echo pytest=$?
for wl in cg cg27; do for dm in 1 2 1 2; do
echo "wl=$wl dot=$dm" >> gpurun_out/ab.log
AOL_LOOP_DOT=$dm AOL_LOOP_TIME=1 DIAG_REPS=4 DIAG_WL=$wl python tools/diag_cg.py >> gpurun_out/ab.log 2>&1
done; done
for bo in 0 64 128; do echo "backoff=$bo" >> gpurun_out/ab.log; AOL_LOOP_BACKOFF_NS=$bo AOL_LOOP_TIME=1 DIAG_REPS=3 python tools/diag_cg.py >> gpurun_out/ab.log 2>&1; done
AOL_LOOP_PROFILE=1 DIAG_REPS=2 python tools/diag_cg.py > gpurun_out/cgprof.log 2>&1
