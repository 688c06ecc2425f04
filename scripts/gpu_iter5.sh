for u in 0.01 0.5; do timeout 120 python scripts/c1_check.py 0 $u; timeout 120 python scripts/c1_check.py 1 $u; done > gpurun_out/it5_c1.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/it5_pytest.log
timeout 600 python scripts/probe.py c2 c4s > gpurun_out/it5_probe.jsonl 2> gpurun_out/it5_probe.err
