"""Per-kernel share of GPU time from an ncu launch list (--metrics gpu__time_duration.sum --csv).
   python tools/launch_shares.py launches.csv"""
import csv
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.reader(lines))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    if r[ui] == "us":
        v *= 1e3
    elif r[ui] == "ms":
        v *= 1e6
    tot[r[ki]] += v
    cnt[r[ki]] += 1
all_ = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / all_ * 100:6.2f}%  {v / cnt[k] / 1e3:9.1f} us avg  x {cnt[k]:4d}  {k[:110]}")
