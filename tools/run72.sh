timeout 600 python tools/e2e_steps.py 2>&1 | tail -8
