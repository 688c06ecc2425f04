set -x
for v in 1 0; do for fill in "" 255; do echo "variant=$v fill=$fill"; KEP_DEBUG_FILL=$fill timeout 120 python scripts/c1_check.py $v 0.5; done; done > gpurun_out/it3_det.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/it3_pytest.log; echo pytest=$?
timeout 600 python scripts/probe.py c2 c4s > gpurun_out/it3_probe.jsonl 2> gpurun_out/it3_probe.err; echo probe=$?
