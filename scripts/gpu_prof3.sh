timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_l21 --launch-skip 20 --launch-count 1 -o gpurun_out/p3_l21 python scripts/prof_run.py 10x10x400 > gpurun_out/p3_a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fsu --launch-skip 300 --launch-count 1 -o gpurun_out/p3_fsu python scripts/prof_run.py 10x10x400 > gpurun_out/p3_b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fsp --launch-skip 300 --launch-count 1 -o gpurun_out/p3_fsp python scripts/prof_run.py 10x10x400 > gpurun_out/p3_c.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p3_launches.csv python scripts/prof_run.py 10x10x400 > gpurun_out/p3_d.log 2>&1
