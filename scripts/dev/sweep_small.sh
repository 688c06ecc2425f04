#!/bin/bash
# k_small thread-count sweep on c4 (dev)
for th in "64,128,128,128,256,256,256,256" "32,64,64,128,128,256,256,256" "128,128,128,256,256,256,256,256"; do
  echo "== $th"; KEP_SMALL_TH=$th python scripts/dev/prof_levels.py 4 8 2 2>&1 | grep -E "shifts/s|L 0|L 1 |L 2|L 3|L 4|L 5"
done
