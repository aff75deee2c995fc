#!/bin/bash
# One-sided pair solve evaluation on the GPU box: eig tests, eig_sym timings per
# SVDK_JACOBI_OS (warps of the one-sided solve; 0 = two-sided solve_pair) and
# SVDK_JACOBI_NS, and the clock64 stamps of a -DSVDK_PROBES build (tools/exp_pair.sh 0).
# usage: tools/jacobi_os_eval.sh [sizes...]   (writes gpurun_out/os_*)
sizes=${@:-256 512 1024 2048}
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "eig or jacobi" > gpurun_out/os_tests.log 2>&1
echo "RC $?" >> gpurun_out/os_tests.log
for cfg in "0 0" "4 1" "4 0" "8 0"; do
  set -- $cfg
  echo "OS=$1 NS=$2" > gpurun_out/os_time_$1_$2.log
  SVDK_JACOBI_OS=$1 SVDK_JACOBI_NS=$2 timeout 300 python tools/eig_time.py $sizes >> gpurun_out/os_time_$1_$2.log 2>&1
done
if [ -f build/exp0/libsvdk.so ]; then
  for w in 4 8; do
    SVDK_JACOBI_OS=$w SVDK_LIB=build/exp0/libsvdk.so timeout 300 python tools/os_probe.py 1024 > gpurun_out/os_probe_$w.log 2>&1
  done
fi
tail -2 gpurun_out/os_tests.log; for f in gpurun_out/os_time_*.log; do head -1 $f; tail -n1 $f; done; tail -n3 gpurun_out/os_probe_*.log
