set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/it2_pytest.log; echo pytest=$?
for v in 0 1; do timeout 300 compute-sanitizer --tool initcheck python scripts/c1_check.py $v 0.5 > gpurun_out/it2_init_$v.log 2>&1; echo init$v=$?; done
timeout 300 compute-sanitizer --tool racecheck python scripts/c1_check.py 0 0.5 > gpurun_out/it2_race_0.log 2>&1; echo race=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_front -s 22 -c 1 -o gpurun_out/it2_front python scripts/prof_run.py > gpurun_out/it2_ncu.log 2>&1; echo ncu=$?
