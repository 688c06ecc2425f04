timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fsp --launch-skip 120 --launch-count 1 -o gpurun_out/p5_fsp python scripts/prof_run.py 10x10x400 > gpurun_out/p5_a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fsp --launch-skip 30 --launch-count 1 -o gpurun_out/p5_fsp2 python scripts/prof_run.py 10x10x400 > gpurun_out/p5_b.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p5_launches.csv python scripts/prof_run.py 10x10x400 > gpurun_out/p5_c.log 2>&1
