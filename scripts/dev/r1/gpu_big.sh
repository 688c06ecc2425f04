timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/big_pytest.log
timeout 1500 python scripts/probe.py c3 > gpurun_out/big_c3.jsonl 2> gpurun_out/big_c3.err
