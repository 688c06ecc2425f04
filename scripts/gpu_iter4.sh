KEP_DEBUG=1 timeout 120 python scripts/c1_check.py 0 0.01 2>&1 | grep -v "batch m=" | head -30
KEP_DEBUG=1 timeout 120 python scripts/c1_check.py 0 0.5 2>&1 | grep -v "batch m=" | tail -4
