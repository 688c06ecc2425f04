# Round-1 final evidence: GPU tests, bench line, launch list of the bench command,
# DRAM traffic of every k_schur launch of one bench step, ncu --set full of one
# k_schur / k_l21<2> / k_assemble launch (c4).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final_ncu_launch.log 2>&1; echo launches=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:'k_schur\(' -c 36 -o gpurun_out/final_schur_all python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/final_ncu_schur_all.log 2>&1; echo schur_all=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_schur\(' --launch-skip 8 -c 1 -o gpurun_out/final_schur_full python scripts/prof_c4.py > gpurun_out/final_ncu_schur_full.log 2>&1; echo schur_full=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_l21<\(int\)2>' --launch-skip 6 -c 3 -o gpurun_out/final_l21_full python scripts/prof_c4.py > gpurun_out/final_ncu_l21_full.log 2>&1; echo l21_full=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assemble --launch-skip 8 -c 1 -o gpurun_out/final_asm_full python scripts/prof_c4.py > gpurun_out/final_ncu_asm_full.log 2>&1; echo asm_full=$?
ls -la gpurun_out/
