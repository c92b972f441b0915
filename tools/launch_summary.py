"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv):
python tools/launch_summary.py launches.csv "title line" > profiles/..._launch_summary.txt"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
h = rows[hdr]
ki, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    v *= scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0].replace("void ", "").replace("mrb::", "")
    tot[name] += v
    cnt[name] += 1
all_t = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print("cold-cache, serialised launches: compare shares, not absolute times")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:45s} n={cnt[k]:5d} total={tot[k]:11.1f} us avg={tot[k] / cnt[k]:10.2f} us "
          f"share={tot[k] / all_t:.3f}")
