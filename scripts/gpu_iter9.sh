for u in 0.01 0.5; do timeout 120 python scripts/c1_check.py 0 $u; done > gpurun_out/it9_c1.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/it9_pytest.log
timeout 600 python scripts/probe.py c2 c4s > gpurun_out/it9_probe.jsonl 2> gpurun_out/it9_probe.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it9_launches.csv python scripts/prof_run.py 10x10x400 > gpurun_out/it9_ncu_launch.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
