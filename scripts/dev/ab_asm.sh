#!/bin/bash
python -m pytest tests/test_gpu_parity.py tests/test_gpu_factor.py -x -q -k "not full_size" 2>&1 | tail -1
for v in "" "KEP_NO_ASM_SMEM=1"; do
  echo "== $v"; env $v python scripts/dev/prof_levels.py 4 8 2 2>&1 | grep -E "shifts/s|^\{'ass|\[kep\] L" | awk '{print $1,$2,$3,$4}'
done
python scripts/dev/prof_levels.py 3 8 1 2>&1 | grep -E "shifts/s"
