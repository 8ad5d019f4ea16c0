for r in 1024 2048 3072 4096 2048 3072; do echo "rows0=$r"; AOL_GEMM2D_ROWS0=$r timeout 300 python tools/probe_e2e_timeline.py 2>&1 | head -3; done
