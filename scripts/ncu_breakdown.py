"""Per-function and per-execution-class instruction breakdown of an ncu source export.
usage: python scripts/ncu_breakdown.py gpurun_out/prof_x [units]   (units = e.g. row-E count)"""
import csv, gzip, sys
from collections import defaultdict
rows = list(csv.reader(gzip.open(sys.argv[1] + ".source.csv.gz", "rt")))
h = rows[1]; rows = rows[2:]
U = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
idx = {n: i for i, n in enumerate(h)}
names = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
tot = {n: sum(int(r[idx[n]] or 0) for r in rows) for n in names}
s = sum(tot.values())
print("stalls:", " ".join(f"{n[6:]}={v / s * 100:.1f}%" for n, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
T = sum(int(r[5]) for r in rows); S = sum(int(r[2]) for r in rows)
print(f"instructions {T:.3e}  per unit {T / U:.1f}")
seg = []; cur = [0, 0, None]
for i, r in enumerate(rows):
    if cur[2] is None: cur[2] = i
    cur[0] += int(r[5]); cur[1] += int(r[2])
    if "RET" in r[1]: seg.append(cur + [i]); cur = [0, 0, None]
seg.append(cur + [len(rows) - 1])
for c in seg:
    if c[0] / T > 0.005:
        print(f"  fn {c[2]:6d}-{c[3]:6d} inst {c[0] / T * 100:5.1f}% ({c[0] / U:7.1f}/unit) samples {c[1] / S * 100:5.1f}%  {rows[c[2]][1].strip()[:40]}")
agg = defaultdict(lambda: [0, 0, 10**9])
for i, r in enumerate(rows):
    c = int(r[5])
    if c: agg[c][0] += 1; agg[c][1] += c; agg[c][2] = min(agg[c][2], i)
print("execution classes:")
for c, (n, sm, first) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
    print(f"  exec/unit {c / U:7.3f} n_instr={n:4d} per_unit={sm / U:7.1f}  first@{first} {rows[first][1].strip()[:40]}")
