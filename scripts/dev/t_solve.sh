#!/bin/bash
python -m pytest tests/test_gpu_factor.py tests/test_gpu_parity.py tests/test_gpu_kth.py -x -q -s -k "not full_size" 2>&1 | tail -4
python scripts/dev/solve_probe.py 2>&1 | grep -E "solves|kth"
python scripts/dev/prof_levels.py 5 2 1 2>&1 | grep -E "shifts/s"
python scripts/dev/prof_levels.py 3 8 1 2>&1 | grep -E "shifts/s"
