timeout 600 python -m pytest tests -m gpu -q -x -k "cg or loop or CG or persistent" > gpurun_out/t_cgfuse.log 2>&1; echo tests=$?
for i in 1 2; do
for f in 0 1; do AOL_LOOP_FUSE=$f AOL_LOOP_TIMING=1 timeout 300 python bench.py --workload cg --steps 10 --warmup 3 --no-e2e --no-cpu --no-peak 2> gpurun_out/cgf_$f.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cg fuse=$f', round(d['value'],1), d['ms_per_step'])"; grep -m1 "us/iter" gpurun_out/cgf_$f.err; done
for f in 0 1; do AOL_LOOP_FUSE=$f AOL_LOOP_TIMING=1 timeout 300 python bench.py --workload cg27 --steps 10 --warmup 3 --no-e2e --no-cpu --no-peak 2> gpurun_out/cg27f_$f.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cg27 fuse=$f', round(d['value'],1), d['ms_per_step'])"; grep -m1 "us/iter" gpurun_out/cg27f_$f.err; done
done
AOL_LOOP_PROFILE=1 timeout 300 python bench.py --workload cg --steps 3 --warmup 3 --no-e2e --no-cpu --no-peak > /dev/null 2> gpurun_out/cg_prof_fused.err
