"""e2e host-path sweep: sogk_sample_host on cfg2 objects with host threads / expansion settings.
   python tools/e2e_sweep.py   (env SOGK_HOST_EXPAND / SOGK_HOST_THREADS are read once per process)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_10272_b200 as P  # noqa: E402

workers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = bench.Workload("cfg2", bench.ProductGen(P))
smp = [P.Sampler([P.build_sparse(d) for d in wl.dense_levels(P, o)], P.Analyzer.hdda, P.KernelKind.skip,
                 wl.step_schedule(P)) for o in range(8)]
rays = [torch.empty((640000, 8), dtype=torch.float64, pin_memory=True) for _ in range(8)]
for o in range(8):
    rays[o].copy_(wl.device_rays(P, 3, o).cpu())
cap = 40_000_000
outs = [dict(pi=torch.empty((640000, 2), dtype=torch.int64, pin_memory=True).numpy(),
             ts=torch.empty(cap, dtype=torch.float64, pin_memory=True).numpy(),
             te=torch.empty(cap, dtype=torch.float64, pin_memory=True).numpy(),
             ri=torch.empty(cap, dtype=torch.int32, pin_memory=True).numpy(),
             st=np.zeros(8, np.int64)) for _ in range(workers)]
from concurrent.futures import ThreadPoolExecutor  # noqa: E402

pool = ThreadPoolExecutor(workers)


def job(w):
    o_ = outs[w]
    for o in range(w, 8, workers):
        P._check(P.lib.sogk_sample_host(smp[o]._h, rays[o].data_ptr(), 640000, 0, cap, o_["pi"].ctypes.data,
                                        o_["ts"].ctypes.data, o_["te"].ctypes.data, o_["ri"].ctypes.data,
                                        None, None, None, None, o_["st"].ctypes.data, None), "host")


for rep in range(4):
    t0 = time.perf_counter()
    list(pool.map(job, range(workers)))
    dt = time.perf_counter() - t0
print(f"workers={workers} expand={os.environ.get('SOGK_HOST_EXPAND', '1')} threads={os.environ.get('SOGK_HOST_THREADS', 'auto')} "
      f"{5.12e6 / dt / 1e6:.1f} Mrays/s ({dt * 1e3:.1f} ms per 8 objects)", flush=True)
