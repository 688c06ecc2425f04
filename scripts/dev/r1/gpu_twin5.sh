timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "twin_c5" 2>&1 | tail -5 > gpurun_out/twin5.log
