timeout 600 python tools/parity/race_probe.py 2>&1 | tail -25
