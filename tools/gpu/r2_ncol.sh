for i in 1 2; do
for w in 0 64 128 192; do
  if [ $w = 0 ]; then AOL_GEMM_NARROW=0 timeout 300 python tools/time_streamk.py 1 2>&1 | sed "s/^/w=256 /";
  else AOL_GEMM_NARROW_ALL=$w timeout 300 python tools/time_streamk.py 1 2>&1 | sed "s/^/w=$w /"; fi
done; done
