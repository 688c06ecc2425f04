set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 200 python scripts/prof_run.py > gpurun_out/r1c4_plain.log 2>&1; echo plain=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1c4_launches.csv python scripts/prof_run.py > gpurun_out/r1c4_ncu_launch.log 2>&1; echo ncu4=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_panel -s 20 -c 2 -o gpurun_out/r1c4_panel python scripts/prof_run.py > gpurun_out/r1c4_ncu_panel.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_schur -s 20 -c 2 -o gpurun_out/r1c4_schur python scripts/prof_run.py > gpurun_out/r1c4_ncu_schur.log 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_assemble -s 20 -c 1 -o gpurun_out/r1c4_asm python scripts/prof_run.py > gpurun_out/r1c4_ncu_asm.log 2>&1; echo ncu3=$?
