for u in 0.01 0.5; do timeout 120 python scripts/c1_check.py 0 $u; done > gpurun_out/it8_c1.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/it8_pytest.log
timeout 600 python scripts/probe.py c2 c4s > gpurun_out/it8_probe.jsonl 2> gpurun_out/it8_probe.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it8_launches.csv python scripts/prof_run.py 10x10x400 > gpurun_out/it8_ncu_launch.log 2>&1
