set -x
timeout 300 python tools/gemm_ncu_probe.py > gpurun_out/gemm_probe2.log 2>&1; cat gpurun_out/gemm_probe2.log
timeout 900 python -m pytest tests/test_gpu_guard.py tests/test_gpu_kernels.py -q -x > gpurun_out/t8.log 2>&1; echo "t8 rc=$?"; tail -3 gpurun_out/t8.log
