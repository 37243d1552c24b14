timeout 600 python tools/e2e_parts.py 2>&1 | tail -12
