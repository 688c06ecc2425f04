#!/bin/bash
# Round-2 ncu --set full captures missing from profiles/: k_spmv2 (c3 stage 1), k_l21<2>, k_fsp,
# k_schur (cp.async) at c4.  Each under its own timeout; --kill ends the run after the capture.
set -x
O=gpurun_out
python scripts/dev/solve_probe.py > $O/r2g_solve.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmv2 -s 2 -c 1 --kill 1 -o $O/r2g_spmv2 \
    python scripts/dev/solve_probe.py > $O/r2g_ncu0.log 2>&1
KEP_FS_STREAMS=0 python scripts/dev/prof_levels.py 4 8 1 > $O/r2g_pl4.log 2>&1
KEP_FS_STREAMS=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_l21<" -s 30 -c 1 --kill 1 -o $O/r2g_l21x \
    python scripts/dev/prof_levels.py 4 8 1 > $O/r2g_ncu1.log 2>&1
KEP_FS_STREAMS=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fsp -s 330 -c 2 --kill 1 -o $O/r2g_fsp \
    python scripts/dev/prof_levels.py 4 8 1 > $O/r2g_ncu2.log 2>&1
KEP_FS_STREAMS=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_schur\(' -s 4 -c 1 --kill 1 -o $O/r2g_schur \
    python scripts/dev/prof_levels.py 4 8 1 > $O/r2g_ncu3.log 2>&1
ls -la $O/*.ncu-rep
