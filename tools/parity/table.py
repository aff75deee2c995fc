"""Build profiles/r2_parity_table.md from `pytest tests/test_gpu_configs.py -s -q` output (the lines
test_config_parity prints: `<config> <method> {parity dict}` and `... vs reference <method> {dict}`)."""
import ast
import re
import sys

rows = []
for line in open(sys.argv[1]):
    m = re.match(r"^[.sFEx]*(c\w+) (\w+) (vs reference \w+ )?(\{.*\})\s*$", line.strip())
    if not m:
        continue
    cfg, method, vs, d = m.groups()
    d = re.sub(r"np\.(?:float64|int64)\(([^()]*)\)", r"\1", d)
    try:
        p = ast.literal_eval(d)
    except Exception:  # noqa: BLE001
        continue
    label = method + (f" (vs ref. {method})" if vs else "")
    rows.append((cfg, label, p))
print("Full-size parity vs the compiled reference (tests/test_gpu_configs.py, B200, round 2, final build; "
      "tools/parity/table.py). Bars: eig <= 1e-10, K exact, top-K sine <= 1e-8, per-vector sine <= 1e-8 "
      "(relative gap >= 1e-6; clusters as subspaces). \"vectors checked\": per-vector comparisons (128 = sampled; "
      "None = the reference sketch fixture stores only the smaller side of the subspace).\n")
print("| config | method | K / K_ref | eig rel err | top-K sine | worst per-vector sine (gap >= 1e-6) | "
      "worst cluster sine | vectors checked |")
print("|---|---|---|---|---|---|---|---|")
for cfg, label, p in rows:
    print(f"| {cfg} | {label} | {p.get('K')} / {p.get('K_ref')} | {p.get('eig_rel_err', float('nan')):.1e} | "
          f"{p.get('topK_sine', float('nan')):.1e} | {p.get('per_vector_sine', 0.0):.1e} | "
          f"{p.get('cluster_sine', 0.0):.1e} | {p.get('vectors_checked')} |")
