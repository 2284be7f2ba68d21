"""Per-kernel timing of pass 1 (count+scan) and pass 2 (write) per object/variant and
launch mode (SOGK_PERSISTENT=1 persistent threads, 0 one thread per ray).
  python tools/kbench.py [cfg2] [variants] [modes]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_10272_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
variants = (sys.argv[2] if len(sys.argv) > 2 else "hdda_skip,dda_branch").split(",")
modes = (sys.argv[3] if len(sys.argv) > 3 else "0,1").split(",")  # "0", "1", "1r8" (refill_min 8)
wl = bench.Workload(P, cfg)
VAR = {"hdda_skip": (1, 1), "hdda_branch": (1, 0), "dda_branch": (0, 0), "dda_skip": (0, 1)}
n = wl.rays_per_object()
tot = {}
for oi, o in enumerate(wl.objects):
    dense = [P.DenseGrid(t, b) for t, b in o["levels"]]
    vdb = [P.build_sparse(d) for d in dense]
    rays = torch.empty((n, 8), dtype=torch.float64, device="cuda")
    wl.fill_rays(rays, 0, oi, 0, 1)
    line = [f"{o['label'][:28]:28s}"]
    for v in variants:
        an, kk = VAR[v]
        for m in modes:
            os.environ["SOGK_PERSISTENT"] = m.split("r")[0]
            os.environ["SOGK_REFILL"] = m.split("r")[1] if "r" in m else "1"
            s = P.Sampler(vdb if an == 1 else dense, an, kk, wl.schedule, cascade=wl.cascade)
            packed, stats = s.count(rays)
            total = int(stats[0].item())
            out = dict(t_starts=torch.empty(max(total, 1), dtype=torch.float64, device="cuda"),
                       t_ends=torch.empty(max(total, 1), dtype=torch.float64, device="cuda"),
                       ray_indices=torch.empty(max(total, 1), dtype=torch.int32, device="cuda"),
                       cells=torch.empty(max(total, 1), dtype=torch.int32, device="cuda"))
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            cs, ws = [], []
            for rep in range(4):
                ev[0].record()
                s.count(rays, packed_info=packed, stats=stats)
                ev[1].record()
                s.write(rays, packed, total, out=out, levels=False)
                ev[2].record()
                torch.cuda.synchronize()
                if rep:
                    cs.append(ev[0].elapsed_time(ev[1]))
                    ws.append(ev[1].elapsed_time(ev[2]))
            c, w = sum(cs) / len(cs), sum(ws) / len(ws)
            tot[(v, m)] = tot.get((v, m), 0) + c + w
            line.append(f"{v}/{m}: {c:6.3f}+{w:6.3f}")
    print(" | ".join(line), f"samples={total}", flush=True)
print("TOTAL", {f"{k[0]}/{k[1]}": round(x, 3) for k, x in tot.items()})
