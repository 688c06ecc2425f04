#!/bin/bash
# Round-2 evidence on one B200: bench line, ncu launch list of the bench command, ncu --set full
# captures of the main kernels (k_schur_tma at c4, k_small at c4, k_bigp/k_bigu at c3, k_fwd/k_bwd/
# k_spmv2 at c3).  Each ncu run follows a clean run of the same command.
set -x
O=gpurun_out
python bench.py --steps 10 --warmup 3 > $O/r2_bench.json 2> $O/r2_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/r2_launches.log 2>&1
python scripts/dev/prof_levels.py 4 8 1 > $O/r2_pl4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_schur_tma -s 2 -c 1 -o $O/r2_schur_tma \
    python scripts/dev/prof_levels.py 4 8 1 > $O/r2_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_small -s 0 -c 1 -o $O/r2_small_full \
    python scripts/dev/prof_levels.py 4 8 1 > $O/r2_ncu2.log 2>&1
python scripts/dev/prof_levels.py 3 8 1 > $O/r2_pl3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_bigp|k_bigu" -s 20 -c 2 -o $O/r2_big_full \
    python scripts/dev/prof_levels.py 3 8 1 > $O/r2_ncu3.log 2>&1
python scripts/dev/solve_probe.py > $O/r2_solve.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_fwd|k_bwd|k_spmv2" -s 16 -c 3 -o $O/r2_solve_full \
    python scripts/dev/solve_probe.py > $O/r2_ncu4.log 2>&1
tail -3 $O/r2_bench.err; head -c 1500 $O/r2_bench.json
