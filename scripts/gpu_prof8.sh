timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p8_launches.csv python scripts/prof_c4.py > gpurun_out/p8_a.log 2>&1
ls -la gpurun_out/
