for q in 640 384; do KEP_NB32_QMAX=$q timeout 600 python scripts/probe.py c4s > gpurun_out/nb_$q.jsonl 2>/dev/null; done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/nb_pytest.log
KEP_NB32_QMAX=384 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/nb_bench384.json 2>/dev/null
