"""Fused render_frame vs two-pass (sample -> composite) on one cfg2/cfg1 object view."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_10272_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
wl = bench.Workload(P, cfg)
for oi, o in enumerate(wl.objects[:3] if cfg == "cfg2" else wl.objects):
    kind, seed, count, base = o["scene"]
    scene = P.analytic_scene(kind, base, seed=seed, count=count)
    cam = wl.camera(0, oi, 0, 1)
    for an, k in ((1, 1), (0, 0)):
        dense = [P.DenseGrid(t, b) for t, b in o["levels"]]
        grids = [P.build_sparse(d) for d in dense] if an == 1 else dense
        s = P.Sampler(grids, an, k, wl.schedule, cascade=wl.cascade)
        d = cam.rays_device()
        def fused():
            return P.render_frame(s, scene, cam)
        def two():
            packed, st = s.count(d)
            tot = int(st[0].item())
            ts, *_ = s.write(d, packed, tot, cells=False, levels=False)
            return P.composite(s, scene, d, packed, ts)
        for name, fn in (("fused", fused), ("two-pass", two)):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                fn()
            e1.record()
            torch.cuda.synchronize()
            print(f"{o['label'][:20]:20s} an={an} k={k} {name:8s} {e0.elapsed_time(e1) / 5:.3f} ms (incl. host sync)", flush=True)
