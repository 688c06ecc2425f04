#!/bin/bash
# A/B of k_l21d (KEP_L21D_MAX) at c4, 8 shifts x 2 reps, optional nrelax
NR=${NR:-16}
for dm in "$@"; do
  KEP_L21D_MAX=$dm KEP_NRELAX=$NR timeout 600 python scripts/dev/prof_levels.py 4 8 2 > gpurun_out/l21d_${dm}_nr${NR}.log 2>&1
  echo "l21d_max=$dm nrelax=$NR"; grep -h "shifts/s\|^{'assemble" gpurun_out/l21d_${dm}_nr${NR}.log
done
