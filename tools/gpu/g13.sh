nproc; free -g | head -2
timeout 1500 python tools/parity/gen_check.py c4 full 2>&1 | tail -12
