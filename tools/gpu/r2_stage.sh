for cfg in "16 4" "32 4" "64 4" "8 8" "32 8"; do set -- $cfg
  AOL_STAGE_SLOT_MB=$1 AOL_STAGE_SLOTS=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-peak --e2e-steps 10 > gpurun_out/r2_stage_$1_$2.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_stage_$1_$2.json').read().splitlines()[0]); print('slot $1 MB x $2:', 'e2e', round(d['e2e']['value'],1), 'e2e_numpy', round(d['e2e_numpy']['value'],1), round(d['e2e_numpy']['ms_per_step'],2), 'ms')"
done
python -c "import torch; print('torch threads', torch.get_num_threads())"
