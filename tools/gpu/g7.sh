set -x
timeout 900 python -m pytest tests/test_gpu_guard.py tests/test_gpu_kernels.py -q -k "guard or trajectory" > gpurun_out/t7.log 2>&1; echo "t7 rc=$?"
tail -4 gpurun_out/t7.log
timeout 300 python tools/gemm_ncu_probe.py > gpurun_out/gemm_probe.log 2>&1; cat gpurun_out/gemm_probe.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -c 2 -o gpurun_out/gemm_r2 python tools/gemm_ncu_probe.py 1048576 1024 > gpurun_out/gemm_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/gemm_ncu.log
