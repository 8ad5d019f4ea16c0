for w in stencil downscaler sweep cg; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_${w}_launches.csv python bench.py --workload $w --steps 2 --warmup 3 --no-e2e --no-cpu --no-peak --no-points > /dev/null 2>&1
  echo "$w rc=$?"
done
