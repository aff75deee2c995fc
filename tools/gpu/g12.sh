timeout 600 python tools/parity/center_check.py c4 2>&1 | tail -12
