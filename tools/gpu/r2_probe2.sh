P="1:gaps:1e7 1:gaps:1e8 2:overlap:1e7 2:overlap:1e8 4:overlap:1e7 8:overlap:1e7"
python tools/sweep_probe.py $P > gpurun_out/probe2_base.log 2>&1
for u in 2 4; do for w in 4 8 16; do AOL_S2_U=$u AOL_S2_WAVES=$w python tools/sweep_probe.py 1:gaps:1e7 1:gaps:1e8 > gpurun_out/probe2_s2_u${u}_w${w}.log 2>&1; done; done
AOL_S2_U=1 AOL_S2_WAVES=8 python tools/sweep_probe.py 1:gaps:1e7 1:gaps:1e8 > gpurun_out/probe2_s2_u1_w8.log 2>&1
for kb in 8 16 32; do for nst in 2 3 4; do for cps in 3 8; do AOL_WIN_KB=$kb AOL_WIN_NST=$nst AOL_WIN_CPS=$cps python tools/sweep_probe.py 2:overlap:1e7 2:overlap:1e8 8:overlap:1e7 > gpurun_out/probe2_win_${kb}_${nst}_${cps}.log 2>&1; done; done; done
