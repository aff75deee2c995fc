#!/bin/bash
# ncu --set full of the Jacobi round kernels (host-driven sweeps so ncu sees the launches):
# one fused round kernel at n = 1024 (launch 60: a mid-sweep round, grid 148) and at n = 256,
# and the quad solve + the two 64-wide updates at n = 4096. Writes gpurun_out/jncu_*.
set -x
M="--set full --clock-control none --import-source on"
SVDK_JACOBI_DEVLOOP=0 timeout 600 ncu $M -k regex:jacobi_round_fused -s 60 -c 1 -o gpurun_out/jncu_fused_1024 -f python tools/eig_one.py 1024 > gpurun_out/jncu_fused_1024.log 2>&1
SVDK_JACOBI_DEVLOOP=0 timeout 600 ncu $M -k regex:jacobi_round_fused -s 30 -c 1 -o gpurun_out/jncu_fused_256 -f python tools/eig_one.py 256 > gpurun_out/jncu_fused_256.log 2>&1
SVDK_JACOBI_DEVLOOP=0 timeout 900 ncu $M -k regex:"jacobi_quad_solve_os|jacobi_update_a64|jacobi_update_v64" -s 300 -c 3 -o gpurun_out/jncu_quad_4096 -f python tools/eig_one.py 4096 > gpurun_out/jncu_quad_4096.log 2>&1
for f in fused_1024 fused_256 quad_4096; do
  ncu -i gpurun_out/jncu_$f.ncu-rep --page details --csv > gpurun_out/jncu_$f.details.csv 2>/dev/null
done
ls -la gpurun_out/jncu_*
