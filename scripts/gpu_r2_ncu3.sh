#!/bin/bash
# ncu --set full captures of k_l21<2> and k_schur (cp.async) at c4 on a mid level (one stream)
set -x
O=gpurun_out
export KEP_FS_STREAMS=0
python scripts/dev/prof_levels.py 4 8 1 > $O/r2h_pl4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:^k_l21$' -s 12 -c 1 --kill 1 -o $O/r2h_l21 \
    python scripts/dev/prof_levels.py 4 8 1 > $O/r2h_ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:^k_schur$' -s 4 -c 1 --kill 1 -o $O/r2h_schur \
    python scripts/dev/prof_levels.py 4 8 1 > $O/r2h_ncu2.log 2>&1
ls -la $O/r2h*.ncu-rep
