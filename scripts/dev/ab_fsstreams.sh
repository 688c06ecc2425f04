#!/bin/bash
# A/B: FS-size groups of a level on forked streams with their k_l21 chains (KEP_FS_STREAMS=1, default)
# vs one stream (0); KEP_FS_SPLIT=k cuts single-group levels into k parts
O=gpurun_out
run() { # cfg streams split
  KEP_FS_STREAMS=$2 KEP_FS_SPLIT=$3 python scripts/dev/prof_levels.py $1 8 2 > $O/ab_fss_c$1_$2_$3.log 2>&1
  echo "c$1 streams=$2 split=$3: $(grep -E 'shifts/s' $O/ab_fss_c$1_$2_$3.log)"
}
run 4 0 1; run 4 1 1; run 4 1 2; run 4 1 3; run 4 1 4
run 3 1 1; run 3 1 2
KEP_FS_SPLIT=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_factor.py -m gpu -x -q -k "not full_size" 2>&1 | tail -3
