"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`.
   python tools/sass_hot.py file.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
body = []
for r in rows[2:]:  # first kernel block only
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(h) and r[0] != "Address":
        body.append(r)
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
src = h.index("Source")
tot = sum(float(r[si] or 0) for r in body)
tot_i = sum(float(r[ii] or 0) for r in body)
print(f"total stall samples {tot:.0f}, warp instructions {tot_i:.0f}, {len(body)} SASS lines")
# stall-reason columns
reason_cols = [i for i, c in enumerate(h) if c.startswith("stall_") or "Stall" in c and i != si]
idx = sorted(range(len(body)), key=lambda k: -float(body[k][si] or 0))[:n]
for k in sorted(idx):
    r = body[k]
    print(f"{k:5d} {float(r[si] or 0) / tot * 100:5.1f}% ex={r[ii]:>10s}  {r[src].strip()[:90]}")
