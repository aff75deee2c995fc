#!/bin/bash
# Per-launch durations of the Jacobi round chain (host-driven sweeps so ncu lists the kernels).
# The fused round kernel appears with three grid sizes: k (first of a sweep: solve only),
# k + workers, and workers only (last of a sweep: the updates alone).
n=${1:-1024}
SVDK_JACOBI_DEVLOOP=0 timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:jacobi_ -s 200 -c 140 --csv \
  python tools/eig_one.py $n > gpurun_out/jl_$n.csv 2> gpurun_out/jl_$n.err
python - <<PY | tee gpurun_out/jl_$n.txt
import csv, collections
rows = list(csv.reader(l for l in open("gpurun_out/jl_$n.csv") if l.startswith('"')))
idx = {h: i for i, h in enumerate(rows[0])}
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[r[idx["ID"]]]["k"] = r[idx["Kernel Name"]].split("(")[0].split("::")[-1]
    per[r[idx["ID"]]][r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
agg = collections.defaultdict(list)
for v in per.values():
    agg[(v["k"], int(v.get("launch__grid_size", 0)))].append(v["gpu__time_duration.sum"])
for (k, g), t in sorted(agg.items()):
    print(f"{k:40s} grid {g:5d}  x{len(t):3d}  mean {sum(t)/len(t)/1e3:7.2f} us  min {min(t)/1e3:7.2f}  max {max(t)/1e3:7.2f}")
PY
