#!/bin/bash
# big-front threshold sweep (dev)
for q in 2048 1024 768; do
  echo "== KEP_BIG_Q=$q"
  for a in "4 8 2" "3 8 1" "5 2 1"; do KEP_BIG_Q=$q python scripts/dev/prof_levels.py $a 2>&1 | grep -E "shifts/s"; done
done
