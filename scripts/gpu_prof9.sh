timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assemble --launch-skip 8 --launch-count 1 -o gpurun_out/p9_asm python scripts/prof_c4.py > gpurun_out/p9_a.log 2>&1
ncu -i gpurun_out/p9_asm.ncu-rep --page source --csv --print-source sass > gpurun_out/p9_asm_sass.csv 2>/dev/null
ls -la gpurun_out/
