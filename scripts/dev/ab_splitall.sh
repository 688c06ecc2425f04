#!/bin/bash
# A/B: every cost-model FS group cut in two on forked streams (KEP_FS_SPLIT_ALL=1) vs not; c5 probe
O=gpurun_out
for v in 0 1; do
  KEP_FS_SPLIT_ALL=$v python scripts/dev/prof_levels.py 4 8 2 > $O/ab_sa_c4_$v.log 2>&1
  echo "c4 split_all=$v: $(grep -E 'shifts/s' $O/ab_sa_c4_$v.log)"
done
KEP_FS_SPLIT_ALL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not full_size" 2>&1 | tail -2
timeout 900 python scripts/dev/prof_levels.py 5 2 1 > $O/r2_probe_c5.log 2>&1
grep -E "shifts/s|n_fronts" $O/r2_probe_c5.log
