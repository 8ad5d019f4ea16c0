for gm in 8 4 16 2 8; do
  AOL_GEMM_GROUP_M=$gm timeout 300 python bench.py --steps 400 --warmup 5 --no-e2e --no-cpu > gpurun_out/gm_$gm.json 2>/dev/null
  python - $gm <<'PY'
import json,sys
for l in open(f"gpurun_out/gm_{sys.argv[1]}.json"):
    if l.startswith("{"):
        d=json.loads(l); c=d["clocks"]
        print("gm", sys.argv[1], "value", round(d["value"],1), "sm_mhz", c.get("sm_mhz"), "power", c.get("power_w_median"), "reasons", c.get("reasons"), flush=True)
PY
done
for gm in 2 4 8 16; do
  AOL_GEMM_GROUP_M=$gm timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:k_gemm_tf32_pair -s 3 -c 1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-peak 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | sed "s/^/gm $gm /"
done
