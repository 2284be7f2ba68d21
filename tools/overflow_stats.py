"""Slab-overflow rays per cfg2 object for a few slab sizes (SOGK_SLAB), HDDA skip."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_10272_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = bench.Workload(P, cfg)
n = wl.rays_per_object()
rays = torch.empty((n, 8), dtype=torch.float64, device="cuda")
for cap in (32, 64, 96, 128, 192):
    os.environ["SOGK_SLAB"] = str(cap)
    row = []
    for oi, o in enumerate(wl.objects):
        grids = [P.build_sparse(P.DenseGrid(t, b)) for t, b in o["levels"]]
        s = P.Sampler(grids, 1, 1, wl.schedule, cascade=wl.cascade)
        wl.fill_rays(rays, 0, oi, 0, 1)
        packed, stats = s.count(rays)
        st = stats.cpu().tolist()
        cnt = packed[:, 1]
        row.append(f"{o['label'][:14]}: ovf {st[6]} hit {int((cnt > 0).sum())} max {int(cnt.max())} mean {st[0] / max(1, int((cnt > 0).sum())):.1f}")
    print(cap, "|", " | ".join(row), flush=True)
