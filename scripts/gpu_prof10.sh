timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l21 --launch-skip 24 --launch-count 6 -o gpurun_out/p10_l21 python scripts/prof_c4.py > gpurun_out/p10_a.log 2>&1
ncu -i gpurun_out/p10_l21.ncu-rep --page source --csv --print-source sass > gpurun_out/p10_l21_sass.csv 2>/dev/null
ls -la gpurun_out/
