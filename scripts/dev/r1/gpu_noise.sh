for i in 1 2; do timeout 600 python scripts/probe.py c4s > gpurun_out/noise_$i.jsonl 2>/dev/null; done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/noise_smi.txt
