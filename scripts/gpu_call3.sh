set -x
timeout 120 python scripts/debug_ref.py > gpurun_out/r1c3_debug.log 2>&1; echo debug_rc=$?
timeout 900 python -m pytest tests -m gpu -v -x --timeout 200 -p no:cacheprovider -k "not 0.5-auto-1" > gpurun_out/r1c3_gpu_tests.log 2>&1; echo tests_rc=$?
timeout 300 python scripts/probe.py c2 c4s > gpurun_out/r1c3_probe.log 2>&1; echo probe_rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r1c3_bench.log 2>&1; echo bench_rc=$?
tail -3 gpurun_out/r1c3_gpu_tests.log
