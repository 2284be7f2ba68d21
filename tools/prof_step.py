"""One count+write pass of a config for ncu (warm-up pass first, then the profiled pass).
  ncu ... -k regex:"count_kernel|write_kernel" -s 2 -c 2 python tools/prof_step.py cfg1 hdda_skip
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_10272_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
var = sys.argv[2] if len(sys.argv) > 2 else "hdda_skip"
obj = int(sys.argv[3]) if len(sys.argv) > 3 else 0
wl = bench.Workload(cfg, bench.ProductGen(P))
an, kk = {"hdda_skip": (1, 1), "hdda_branch": (1, 0), "dda_branch": (0, 0), "dda_skip": (0, 1)}[var]
o = wl.objects[obj]
dense = wl.dense_levels(P, obj)
grids = [P.build_sparse(d) for d in dense] if an == 1 else dense
s = P.Sampler(grids, an, kk, wl.step_schedule(P), cascade=wl.cascade, ray_order=wl.ray_order)
rays = wl.device_rays(P, 0, obj)
for it in range(2):
    packed, stats = s.count(rays)
    tot = int(stats[0].item())
    s.write(rays, packed, tot, levels=False)
torch.cuda.synchronize()
print("total samples", tot, "stats", stats.cpu().tolist())
