#!/bin/bash
# A/B of one environment knob at c4 (8 shifts x 2 reps): ab_env.sh VAR v1 v2 ...
VAR=$1; shift
for v in "$@"; do
  env $VAR=$v timeout 600 python scripts/dev/prof_levels.py 4 8 2 > gpurun_out/ab_${VAR}_${v}.log 2>&1
  echo "$VAR=$v"; grep -h "shifts/s\|^{'assemble" gpurun_out/ab_${VAR}_${v}.log | cut -c1-200
done
