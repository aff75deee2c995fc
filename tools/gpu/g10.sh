set -x
timeout 600 python tools/parity/gen_check.py c4 2>&1 | tail -12
timeout 600 python tools/parity/c4_vector_diag.py c4 2>&1 | tail -60
