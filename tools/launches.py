"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    out = []
    for r in rows[1:]:
        if len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
            out.append((r[i_name], float(r[i_val].replace(",", ""))))
    return out


if __name__ == "__main__":
    launches = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, ns in launches:
        key = name.split("(")[0][-70:]
        agg[key][0] += 1
        agg[key][1] += ns
    total = sum(t for _, t in agg.values())
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t / 1e6:10.3f} ms {100 * t / total:5.1f}%  n={c:5d}  avg {t / c / 1e3:9.1f} us  {k}")
