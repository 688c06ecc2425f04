timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
for x in 48 56 64; do KEP_XMIN=$x timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/xmin_$x.json 2> gpurun_out/xmin_$x.err; done
