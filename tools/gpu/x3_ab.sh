for i in 1 2 3; do
AOL_LIB=paper_1105_4424_b200/_lib/libaolb200_smemA.so python tools/time_3xtf32.py | sed 's/^/smemA /'
AOL_LIB=paper_1105_4424_b200/_lib/libaolb200_tmemA.so python tools/time_3xtf32.py | sed 's/^/tmemA /'
done
