"""Pass-1 time with and without ray binning on camera-ray configs (object views of cfg2/cfg1)."""
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
tot = {0: 0.0, 1: 0.0}
for oi, o in enumerate(wl.objects):
    wl.fill_rays(rays, 0, oi, 0, 1)
    dense = [P.DenseGrid(t, b) for t, b in o["levels"]]
    grids = [P.build_sparse(d) for d in dense]
    for order in (0, 1):
        s = P.Sampler(grids, 1, 1, wl.schedule, cascade=wl.cascade, ray_order=order)
        for _ in range(2):
            s.count(rays)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            s.count(rays)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        tot[order] += ms
        print(f"{o['label'][:24]:24s} order={order} count {ms:.3f} ms", flush=True)
print("total", tot)
