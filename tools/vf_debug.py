"""Debug the voxel fast path on the tie rays: traverse events and sample counts vs the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_10272_b200 as P  # noqa: E402
from oracle_bindings import BRANCH, HDDA, SKIP, Oracle  # noqa: E402
from parity_util import gpu_sample, host_grid, oracle_sample  # noqa: E402
from test_gpu_voxel_fast import _tie_rays  # noqa: E402

res = 32
t = P.GridTransform((res, res, res), (0.0, 0.0, 0.0), 1.0)
bits = np.zeros(t.payload_bytes(), np.uint8)
for z in range(res):
    for y in range(res):
        for x in range(res):
            if (x + y + z) % 2 == 0:
                i = (z * res + y) * res + x
                bits[i >> 3] |= 1 << (i & 7)
g = host_grid(P, t, bits)
rays = _tie_rays(res)
O = Oracle()
sched = P.StepSchedule.constant(0.25)
for k in (SKIP, BRANCH):
    got = gpu_sample(P, [g], HDDA, k, sched, rays)
    want = oracle_sample(O, [g], HDDA, k, sched, rays)
    bad = np.nonzero(got.packed_info[:, 1] != want.packed_info[:, 1])[0]
    badc = np.nonzero((got.counters != want.counters).any(axis=1))[0]
    print("kernel", k, "count mismatches", bad.size, bad[:8], "counter mismatches", badc.size, badc[:8])
    for r in bad[:3]:
        print("  ray", r, list(rays[r]), "got", got.packed_info[r], got.counters[r], "want", want.packed_info[r], want.counters[r])
s = P.Sampler([P.build_sparse(P.DenseGrid(t, bits))], HDDA, SKIP, sched)
tr = s.traverse_host(rays)
s2 = O.sampler([g], HDDA, SKIP, 0, 1.0)
nb = 0
for r in range(rays.shape[0]):
    n, ev, c = O.events(s2, rays[r])
    if n < 0:
        if tr.status[r] != 2:
            nb += 1
        continue
    o, cnt = tr.event_info[r]
    e = tr.events[o:o + cnt]
    same = cnt == n and all(tuple(e[j]["ijk"]) == ev[j][0] and e[j]["t0"] == ev[j][2] and e[j]["t1"] == ev[j][3] for j in range(n))
    if not same:
        nb += 1
        if nb <= 3:
            print("event mismatch ray", r, "n", cnt, n)
            for j in range(min(cnt, n)):
                if not (tuple(e[j]["ijk"]) == ev[j][0] and e[j]["t0"] == ev[j][2] and e[j]["t1"] == ev[j][3]):
                    print("   first diff", j, tuple(e[j]["ijk"]), e[j]["t0"], e[j]["t1"], "|", ev[j][0], ev[j][2], ev[j][3])
                    break
print("traverse mismatching rays", nb, "of", rays.shape[0])
