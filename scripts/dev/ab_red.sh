#!/bin/bash
for v in "" "KEP_SCHUR_RED=1"; do
  echo "== $v"; env $v python scripts/dev/prof_levels.py 4 8 2 2>&1 | grep -E "shifts/s|L 0|L 1 |L 2|L 3|L 4"
done
