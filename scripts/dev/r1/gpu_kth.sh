timeout 1200 python -X faulthandler -m pytest tests/test_gpu_kth.py -q -x -p no:cacheprovider > gpurun_out/kth.log 2>&1; echo "exit=$?" >> gpurun_out/kth.log
