DIAG_WL=cg27 DIAG_REPS=1 python tools/diag_cg.py > gpurun_out/p4.log 2>&1 && \
DIAG_WL=cg27 DIAG_REPS=1 ncu --set full --clock-control none --import-source on -k regex:k_loop_persistent -c 1 -o gpurun_out/prof_cg27 python tools/diag_cg.py > gpurun_out/ncu_cg27.log 2>&1
echo a=$?
DIAG_WL=cg DIAG_REPS=1 python tools/diag_cg.py > gpurun_out/p5.log 2>&1 && \
DIAG_WL=cg DIAG_REPS=1 ncu --set full --clock-control none --import-source on -k regex:k_loop_persistent -c 1 -o gpurun_out/prof_cg python tools/diag_cg.py > gpurun_out/ncu_cg.log 2>&1
echo b=$?
