"""Where the grid-build time goes: wall time of build_sparse / build_distance split into the
build call (allocation + launches + any sync), the device time (CUDA events) and the destroy."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2404_10272_b200 as P  # noqa: E402


def probe(kind, res, fn, reps=10):
    t = P.GridTransform.cube(res, (-1.0, -1.0, -1.0), 2.0)
    bits, _ = P.generate_scene(kind, t, seed=1)
    d = P.DenseGrid(t, bits)
    fn(d)  # warm
    torch.cuda.synchronize()
    calls, devs, dels = [], [], []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0.record()
        g = fn(d)
        e1.record()
        w1 = time.perf_counter()
        torch.cuda.synchronize()
        w2 = time.perf_counter()
        del g
        w3 = time.perf_counter()
        calls.append((w1 - w0) * 1e3)
        devs.append(e0.elapsed_time(e1))
        dels.append((w3 - w2) * 1e3)
    med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
    print(f"{fn.__name__:15s} {kind:6s} {res:4d}: call {med(calls):8.3f} ms  events {med(devs):8.3f} ms"
          f"  destroy {med(dels):8.3f} ms")


for res in (128, 256, 512):
    for kind in ("blobs", "shell"):
        probe(kind, res, P.build_sparse)
        probe(kind, res, P.build_distance)
