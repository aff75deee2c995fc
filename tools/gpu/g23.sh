timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_guard.py tests/test_gpu_configs.py -q -x -k "eig or jacobi or c1 or c4 or trajectory" > gpurun_out/t23.log 2>&1; echo "t23 rc=$?"; tail -3 gpurun_out/t23.log
timeout 600 python tools/eig_time.py 256 512 1024 2048 4096 2>&1 | tail -1
