for i in 1 2 3; do
python bench.py --steps 400 --no-cpu --no-peak > gpurun_out/mm_e2e.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/mm_e2e.json')); print(round(d['value'],1), d['e2e'])" >> gpurun_out/e2e_numa.log
done
nproc >> gpurun_out/e2e_numa.log; lscpu | grep -i numa >> gpurun_out/e2e_numa.log
