for t in time_filters time_shift time_blocks time_tile_sum time_stencil_kxk time_exact time_batched; do echo "== $t"; timeout 300 python tools/$t.py 2>&1 | tail -25; done
