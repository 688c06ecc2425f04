timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p12_launches.csv python scripts/prof_c4.py > gpurun_out/p12_a.log 2>&1
