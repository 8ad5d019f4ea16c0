for sp in 1 2 3 4 8; do
  if [ $sp = 1 ]; then E="AOL_GEMM_STREAMK=0"; else E="AOL_GEMM_SPLIT=$sp"; fi
  env $E timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:k_gemm_tf32_pair -s 10 -c 2 --csv --log-file gpurun_out/r2_skd_$sp.csv python tools/time_streamk.py 8 > /dev/null 2>&1
done
for sp in 2 3 4 8; do AOL_GEMM_SPLIT=$sp timeout 300 python tools/time_streamk.py 8 4; done
