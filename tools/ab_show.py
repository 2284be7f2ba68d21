"""Print the per-variant step times of bench JSON lines: python tools/ab_show.py gpurun_out/TAG_*.json"""
import json
import sys

for f in sys.argv[1:]:
    try:
        line = [l for l in open(f) if l.startswith("{")][-1]
        d = json.loads(line)
    except Exception as e:  # noqa: BLE001
        print(f, "no result", e)
        continue
    v = d["variants"]
    print(f"{f:48s} {d['value'] / 1e6:8.1f} Mrays/s  " + "  ".join(
        f"{k}: {x['ms_per_step']:.3f} ({x['count_ms_per_step']:.3f}+{x['write_ms_per_step']:.3f})" for k, x in v.items()))
