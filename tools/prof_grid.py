"""One HDDA count+write pass on a 128^3 grid for ncu (warm-up pass first).
   python tools/prof_grid.py random 0.02 [n_log2]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2404_10272_b200 as P  # noqa: E402

fam, frac = sys.argv[1], float(sys.argv[2])
n = 1 << (int(sys.argv[3]) if len(sys.argv) > 3 else 20)
t = P.GridTransform.cube(128, (-1.0, -1.0, -1.0), 2.0)
bits = P.random_grid(t, 7, frac) if fam == "random" else P.random_blocky_grid(t, 7, frac, 0.001)
s = P.Sampler([P.build_sparse(P.DenseGrid(t, bits))], P.Analyzer.hdda, P.KernelKind.skip,
              P.StepSchedule.constant(0.5 * t.voxel_size))
rays = torch.from_numpy(P.make_probe_rays(t, n, 5)).cuda()
for _ in range(2):
    pk, st = s.count(rays)
    tot = int(st[0].item())
    s.write(rays, pk, tot, levels=False)
torch.cuda.synchronize()
print("samples", tot)
