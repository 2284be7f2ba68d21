"""One cfg1 frame per variant through sogk_render_camera (for an ncu launch list)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_10272_b200 as P  # noqa: E402

wl = bench.Workload("cfg1", bench.ProductGen(P))
o = wl.objects[0]
kind, seed, count = o["scene"]
scene = P.analytic_scene(kind, P.GridTransform(*o["levels"][0][:3]), seed=seed, count=count)
cam = wl.camera(P, wl.shard(0, 0, 0, 1))
dense = wl.dense_levels(P, 0)
for an, k in ((1, 1), (0, 0)):
    grids = [P.build_sparse(d) for d in dense] if an == 1 else dense
    s = P.Sampler(grids, an, k, wl.step_schedule(P))
    for _ in range(3):
        f = P.render_frame(s, scene, cam)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f = P.render_frame(s, scene, cam)
    e1.record()
    torch.cuda.synchronize()
    print(f"an={an} frame {e0.elapsed_time(e1) / 5:.3f} ms samples {f.samples}", flush=True)
