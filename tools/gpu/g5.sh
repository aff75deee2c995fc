set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t5.log 2>&1; echo "t5 rc=$?"
tail -8 gpurun_out/t5.log
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -s -k "trajectory" 2>&1 | grep -E "engine trajectory|passed|failed"
timeout 600 python tools/eig_time.py 256 512 1024 2048 4096 2>&1 | tail -2
