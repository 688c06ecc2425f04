set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -v -x --timeout 150 -p no:cacheprovider > gpurun_out/r1c2_gpu_tests.log 2>&1; echo tests_rc=$?
timeout 300 python scripts/probe.py c1 c2 c4s > gpurun_out/r1c2_probe.log 2>&1; echo probe_rc=$?
timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python __graft_entry__.py > gpurun_out/r1c2_memcheck.log 2>&1; echo memcheck_rc=$?
tail -3 gpurun_out/r1c2_gpu_tests.log
