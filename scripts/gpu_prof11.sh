timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fsp --launch-skip 110 --launch-count 1 -o gpurun_out/p11_fsp python scripts/prof_c4.py > gpurun_out/p11_a.log 2>&1
ncu -i gpurun_out/p11_fsp.ncu-rep --page source --csv --print-source sass > gpurun_out/p11_fsp_sass.csv 2>/dev/null
ls -la gpurun_out/
