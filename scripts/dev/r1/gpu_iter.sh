# quick iteration: GPU tests, probe, short bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/it_pytest.log; echo pytest=$?
timeout 600 python scripts/probe.py c2 c4s > gpurun_out/it_probe.jsonl 2> gpurun_out/it_probe.err; echo probe=$?
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; echo bench=$?
