#!/bin/bash
# Sweep the GEMV-pair cluster size / lookahead on the c3, c5 and c2 shapes
# (plus the automatic choice, "auto").
out=${1:-gpurun_out/gemv_sweep.txt}
rm -f "$out"
for shape in "500000 2048" "65536 4096" "200000 1024" "20000 256"; do
  echo -n "$shape auto: " >> "$out"
  timeout 60 python tools/gemv_probe.py $shape 3 >> "$out" 2>&1
  for cs in ${CS_LIST:-2 4 8}; do
    for la in ${LA_LIST:-0 1}; do
      echo -n "$shape cs=$cs la=$la: " >> "$out"
      SVDK_GEMV_CS=$cs SVDK_GEMV_LA=$la timeout 60 python tools/gemv_probe.py $shape 3 >> "$out" 2>&1
    done
  done
done
