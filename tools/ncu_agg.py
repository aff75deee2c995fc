"""Average per-kernel metrics of an `ncu --csv --metrics ...` launch list."""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
idx = {h: i for i, h in enumerate(rows[0])}
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    k = r[idx["Kernel Name"]].split("(")[0].split("::")[-1]
    agg[k][r[idx["Metric Name"]]].append(float(r[idx["Metric Value"]].replace(",", "")))
for k, m in agg.items():
    n = len(next(iter(m.values())))
    print(k, n, {name.split("__")[-1][:40]: round(sum(v) / len(v), 1) for name, v in m.items()})
