for t in 192 700; do KEP_FSP_TH128=$t timeout 600 python scripts/probe.py c4s c2 > gpurun_out/th_$t.jsonl 2>/dev/null; done
KEP_FSP_TH128=700 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/th_bench700.json 2>/dev/null
