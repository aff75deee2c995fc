timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_guard.py tests/test_gpu_configs.py tests/test_gpu_methods.py -q -x -k "eig or jacobi or c1 or c4 or c2 or trajectory or lanczos or small" > gpurun_out/t24.log 2>&1; echo "t24 rc=$?"; tail -3 gpurun_out/t24.log; grep -E "^E " gpurun_out/t24.log | head -5
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -s -k trajectory 2>&1 | grep "engine trajectory"
echo warp; timeout 600 python tools/eig_time.py 256 512 1024 2048 2>&1 | tail -1
echo cta; SVDK_JACOBI_WARP=0 timeout 600 python tools/eig_time.py 256 512 1024 2048 2>&1 | tail -1
