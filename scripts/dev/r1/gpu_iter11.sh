bash scripts/gpu_iter10.sh
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_l21<\(int\)2>' --launch-skip 8 -c 1 -o gpurun_out/final_l21_full python scripts/prof_c4.py > gpurun_out/final_ncu_l21_full.log 2>&1
