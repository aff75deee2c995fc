#!/bin/bash
# Jacobi tuning sweep: block size TB x inner sweep cap, n in {256, 1024, 2048}
for n in 256 1024 2048; do
  for tb in 16 32 64; do
    for inner in 1 2 3 8; do
      r=$(SVDK_JACOBI_TB=$tb SVDK_JACOBI_INNER=$inner timeout 120 python tools/eig_probe.py $n 2 2>&1 | tail -2 | tr '\n' ' ')
      echo "n=$n TB=$tb inner=$inner :: $r"
    done
  done
done
