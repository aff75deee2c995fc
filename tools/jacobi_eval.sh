#!/bin/bash
# Jacobi scheme evaluation on the GPU box: eig parity tests, eig_sym timings for
# the 2b = 32 and quad (64) schemes, per-kernel launch times at n = 4096.
# usage: tools/jacobi_eval.sh [sizes...]   (writes gpurun_out/jeval_*)
sizes=${@:-256 512 1024 2048 4096}
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k eig > gpurun_out/jeval_tests.log 2>&1
echo "RC $?" >> gpurun_out/jeval_tests.log
for tb in 32 64; do
  SVDK_JACOBI_TB=$tb timeout 300 python tools/eig_time.py $sizes > gpurun_out/jeval_time_$tb.log 2>&1
done
SVDK_JACOBI_TB=64 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:jacobi_ -s 300 -c 30 --csv python tools/eig_probe.py 4096 > gpurun_out/jeval_launch.csv 2> gpurun_out/jeval_launch.err
