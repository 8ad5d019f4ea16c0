for b in 0 8 32 64 128; do echo "backoff $b"; AOL_LOOP_BACKOFF_NS=$b AOL_LOOP_TIME=1 DIAG_REPS=3 timeout 300 python tools/diag_cg.py graphs 2>&1 | grep -E "graphs:|kernel" | tail -2; done
for b in 0 32; do echo "cg27 backoff $b"; DIAG_WL=cg27 AOL_LOOP_BACKOFF_NS=$b AOL_LOOP_TIME=1 DIAG_REPS=3 timeout 300 python tools/diag_cg.py graphs 2>&1 | grep -E "graphs:|kernel" | tail -2; done
