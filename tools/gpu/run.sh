python bench.py --steps 100 --no-cpu > gpurun_out/mm.json 2>/dev/null; echo mm=$?
