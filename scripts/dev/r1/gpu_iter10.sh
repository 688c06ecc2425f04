for u in 0.01 0.5; do timeout 120 python scripts/c1_check.py 0 $u; done > gpurun_out/it10_c1.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/it10_pytest.log
timeout 600 python scripts/probe.py c2 c4s > gpurun_out/it10_probe.jsonl 2> gpurun_out/it10_probe.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err
