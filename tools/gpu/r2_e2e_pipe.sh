for p in 8 16 32 8 16 32; do AOL_E2E_PIPELINE=$p timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-peak --no-e2e-numpy --e2e-steps 20 > gpurun_out/r2_e2e_p$p.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r2_e2e_p$p.json').read().splitlines()[0]); print('pipeline $p', round(d['e2e']['value'],2), round(d['e2e']['ms_per_step'],3))"; done
