python -m pytest tests/test_gpu_parity.py -x -q -k "cg or loop or dot" > gpurun_out/pytest_cg.log 2>&1; echo pytest=$?
for wl in cg cg27; do for f in 0 1 0 1; do
echo "wl=$wl fuse=$f" >> gpurun_out/ab.log
AOL_LOOP_FUSE_SCALARS=$f AOL_LOOP_TIME=1 DIAG_REPS=4 DIAG_WL=$wl python tools/diag_cg.py >> gpurun_out/ab.log 2>&1
done; done
