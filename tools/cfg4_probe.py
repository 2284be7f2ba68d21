"""cfg4 pass-2 variance probe: overflow rays, run counts, and per-kernel times of a few steps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_10272_b200 as P  # noqa: E402

wl = bench.Workload(P, "cfg4")
o = wl.objects[0]
dense = [P.DenseGrid(t, b) for t, b in o["levels"]]
grids = [P.build_sparse(d) for d in dense]
s = P.Sampler(grids, 1, 1, wl.schedule)
n = wl.rays_per_object()
rays = torch.empty((n, 8), dtype=torch.float64, device="cuda")
for step in range(4):
    wl.fill_rays(rays, step, 0, 0, 1)
    packed, stats = s.count(rays)
    st = stats.cpu().tolist()
    cnt = packed[:, 1]
    tot = int(st[0])
    out = dict(t_starts=torch.empty(tot, dtype=torch.float64, device="cuda"),
               t_ends=torch.empty(tot, dtype=torch.float64, device="cuda"),
               ray_indices=torch.empty(tot, dtype=torch.int32, device="cuda"),
               cells=torch.empty(tot, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.write(rays, packed, tot, out=out, levels=False)
    e1.record()
    torch.cuda.synchronize()
    print(f"step {step}: total {tot} overflow rays {st[6]} max count {int(cnt.max())} write {e0.elapsed_time(e1):.3f} ms", flush=True)
