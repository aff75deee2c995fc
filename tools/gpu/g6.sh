set -x
timeout 900 python -m pytest tests/test_gpu_guard.py -q > gpurun_out/t6a.log 2>&1; echo "guard rc=$?"
tail -15 gpurun_out/t6a.log
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_kernels.py -q -s -k "c4 or trajectory or c2mid or c1" > gpurun_out/t6b.log 2>&1; echo "cfg rc=$?"
grep -E "c4|c2mid|c1 |trajectory|passed|failed" gpurun_out/t6b.log | tail -20
