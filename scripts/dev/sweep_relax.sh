#!/bin/bash
# nrelax / relax_frac sweep at c4 (8 shifts, 2 reps): per-level profile per setting
for x in "$@"; do
  nr=${x%:*}; fr=${x#*:}
  KEP_NRELAX=$nr KEP_RELAX_FRAC=$fr timeout 600 python scripts/dev/prof_levels.py 4 8 2 > gpurun_out/relax_${nr}_${fr}.log 2>&1
  grep -h "shifts/s\|flops_exec" gpurun_out/relax_${nr}_${fr}.log
done
