timeout 600 python scripts/probe.py c2 c4s > gpurun_out/pr_probe.jsonl 2> gpurun_out/pr_probe.err
