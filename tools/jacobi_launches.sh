#!/bin/bash
# Per-kernel durations of the Jacobi round chain (host-driven sweeps so ncu lists the kernels).
n=${1:-1024}
SVDK_JACOBI_DEVLOOP=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:jacobi_ -s 400 -c 120 --csv \
  python tools/eig_one.py $n > gpurun_out/jl_$n.csv 2> gpurun_out/jl_$n.err
python tools/ncu_agg.py gpurun_out/jl_$n.csv | tee gpurun_out/jl_$n.txt
