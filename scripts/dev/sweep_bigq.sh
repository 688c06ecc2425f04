#!/bin/bash
# big-front threshold sweep (dev)
for q in 3072 4096 8192; do
  echo "== KEP_BIG_Q=$q"
  for a in "3 8 1" "5 2 1"; do KEP_BIG_Q=$q python scripts/dev/prof_levels.py $a 2>&1 | grep -E "shifts/s"; done
done
