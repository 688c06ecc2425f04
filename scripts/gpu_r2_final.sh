#!/bin/bash
# Round-2 final evidence at HEAD on one B200: per-level profile (c4), ncu launch list of the bench
# command, ncu --set full captures of k_l21<2>, k_fsp, k_schur (cp.async), k_l21d at c4.
# Each ncu run follows a clean run of the same command.
set -x
O=gpurun_out
python scripts/dev/prof_levels.py 4 8 2 > $O/r2f_pl4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2f_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/r2f_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_l21<2>|k_l21<\(int\)2>" -s 6 -c 1 -o $O/r2f_l21x \
    python scripts/dev/prof_levels.py 4 8 1 > $O/r2f_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fsp -s 200 -c 2 -o $O/r2f_fsp \
    python scripts/dev/prof_levels.py 4 8 1 > $O/r2f_ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_schur$|k_l21d" -s 4 -c 3 -o $O/r2f_schur_l21d \
    python scripts/dev/prof_levels.py 4 8 1 > $O/r2f_ncu3.log 2>&1
tail -25 $O/r2f_pl4.log
