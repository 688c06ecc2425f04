timeout 900 python -m pytest tests/test_gpu_kth.py -q -x -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/c5_kth.log
KEP_DEBUG=1 timeout 2400 python scripts/probe.py c5 > gpurun_out/c5_probe.jsonl 2> gpurun_out/c5_probe.err
