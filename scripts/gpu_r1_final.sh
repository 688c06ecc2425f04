set -x
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final_ncu_launch.log 2>&1; echo launches=$?
timeout 1200 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --clock-control none -k regex:k_schur -c 20 -o gpurun_out/final_schur_all python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/final_ncu_schur_all.log 2>&1; echo schur_all=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_schur --launch-skip 8 -c 1 -o gpurun_out/final_schur_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/final_ncu_schur_full.log 2>&1; echo schur_full=$?
