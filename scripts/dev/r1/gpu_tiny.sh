for t in 0 24 40; do KEP_TINY_REF=$t timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tiny_$t.json 2> gpurun_out/tiny_$t.err; done
KEP_TINY_REF=40 timeout 300 python scripts/c1_check.py 0 0.01 > gpurun_out/tiny_c1.log 2>&1
