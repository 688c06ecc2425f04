timeout 900 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f1_full.log 2>&1; echo "exit=$?" >> gpurun_out/f1_full.log
