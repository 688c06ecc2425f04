#!/bin/bash
# per-level A/B of the TMA Schur kernel (dev)
for v in "" "KEP_NO_TMA=1"; do
  echo "== $v"; env $v python scripts/dev/prof_levels.py 4 8 2 2>&1 | grep -E "shifts/s|schur TF|\[kep\] L" | awk '{print $1, $2, $3, $7}'
done
for v in "" "KEP_NO_TMA=1"; do
  echo "== c5 $v"; env $v python scripts/dev/prof_levels.py 5 2 1 2>&1 | grep -E "shifts/s|schur TF|\[kep\] L" | awk '{print $1, $2, $3, $7}'
done
