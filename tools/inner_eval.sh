#!/bin/bash
# Block-Jacobi variants: inner sweeps per pair solve x split/full scheme (timing + sweeps).
sizes=${@:-1024 2048}
for sch in split full; do for inner in 1 2 3; do
  echo "scheme=$sch inner=$inner" 
  SVDK_JACOBI_SCHEME=$sch SVDK_JACOBI_INNER=$inner timeout 300 python tools/eig_time.py $sizes 2>&1 | tail -1
done; done > gpurun_out/inner_eval.log 2>&1
cat gpurun_out/inner_eval.log
