timeout 600 python tools/parity/gram_check.py c4 2>&1 | tail -12
