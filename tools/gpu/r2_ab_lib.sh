# same box: the pre-mixed-width library vs the current one, alternated, 8192^3 and the 8-rank shard
for i in 1 2 3; do
  AOL_LIB=_ab/libaolb200_pre_narrow.so timeout 300 python tools/time_streamk.py 1 8 2>&1 | sed "s/^/pre  /"
  timeout 300 python tools/time_streamk.py 1 8 2>&1 | sed "s/^/now  /"
done
