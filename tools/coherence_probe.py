"""Does reordering incoherent probe rays by (entry cell, direction) speed up pass 1? (cfg4)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_10272_b200 as P  # noqa: E402

wl = bench.Workload(P, "cfg4")
o = wl.objects[0]
t, bits = o["levels"][0]
dense = P.DenseGrid(t, bits)
grids = {1: [P.build_sparse(dense)], 2: [P.build_distance(dense)], 0: [dense]}
h = P.make_probe_rays(t, 1 << 24, seed=1000)
o_, d_ = h[:, :3], h[:, 3:6]
# entry point into the grid box [-1, 1]^3 (slab clip), coarse cell + direction octant key
with np.errstate(divide="ignore", invalid="ignore"):
    ta = (-1.0 - o_) / d_
    tb = (1.0 - o_) / d_
te = np.nanmax(np.minimum(ta, tb), axis=1).clip(min=0.0)
ent = o_ + d_ * te[:, None]
q = np.clip(((ent + 1.0) * 8).astype(np.int64), 0, 15)          # 16^3 entry cells
oc = (d_ > 0).astype(np.int64) @ np.array([1, 2, 4])               # direction octant
dq = np.clip(((d_ + 1.0) * 4).astype(np.int64), 0, 7)             # 8^3 direction cells
key = (((q[:, 0] * 16 + q[:, 1]) * 16 + q[:, 2]) * 512 + (dq[:, 0] * 8 + dq[:, 1]) * 8 + dq[:, 2]) * 8 + oc
order = np.argsort(key, kind="stable")
for name, arr in (("original", h), ("sorted", h[order])):
    d = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
    for an, k in ((1, 1), (2, 1), (0, 0)):
        s = P.Sampler(grids[an], an, k, wl.schedule)
        for _ in range(2):
            s.count(d)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            s.count(d)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:9s} an={an} count {e0.elapsed_time(e1) / 3:.2f} ms", flush=True)
