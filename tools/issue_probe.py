"""Pass-1 issue ceiling input: warp instructions of count_kernel for one bench step.

pass 1 (count_kernel) is bound by instruction issue, not HBM, so bench.py
reports its issue-slot fraction beside the HBM roofline: warp instructions per step (this
capture) / pass-1 time (live) / (148 SMs x 4 schedulers x SM clock).

    ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none \
        -k regex:count_kernel --csv --log-file gpurun_out/issue_cfg2.csv \
        python tools/issue_probe.py run cfg2
    python tools/issue_probe.py parse cfg2 gpurun_out/issue_cfg2.csv   # -> profiles/issue_cfg2.json
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

STEP = 3  # the first timed step of the default bench run (--warmup 3)


def run(cfg):
    import torch

    import bench
    import paper_2404_10272_b200 as P

    wl = bench.Workload(cfg, bench.ProductGen(P))
    n = wl.rays_per_object()
    for obj, o in enumerate(wl.objects):
        grids = [P.build_sparse(d) for d in wl.dense_levels(P, obj)]
        s = P.Sampler(grids, P.Analyzer.hdda, P.KernelKind.skip, wl.step_schedule(P), cascade=wl.cascade,
                      ray_order=wl.ray_order)
        rays = wl.device_rays(P, STEP, obj)
        for _ in range(2):  # warm launch, then the one that is kept
            s.count(rays)
        torch.cuda.synchronize()
    print("objects", len(wl.objects), "rays per object", n)


def parse(cfg, path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ii = h.index("ID")
    launches = {}
    for r in rows[1:]:
        if len(r) <= vi or "count_kernel<" not in r[ki]:  # not bin_count_kernel
            continue
        launches.setdefault(int(r[ii]), {})[r[mi]] = float(r[vi].replace(",", ""))
    ids = sorted(launches)
    kept = [launches[i] for i in ids[1::2]]  # the second launch of every object
    inst = sum(k["smsp__inst_executed.sum"] for k in kept)
    ns = sum(k["gpu__time_duration.sum"] for k in kept)
    out = {"config": cfg, "variant": "sparse+hdda+skip", "step": STEP, "launches": len(kept),
           "pass1_warp_inst_per_step": inst, "ncu_count_kernel_ns_per_step": ns,
           "source": f"ncu smsp__inst_executed.sum of count_kernel, tools/issue_probe.py ({path})"}
    dst = os.path.join(ROOT, "profiles", f"issue_{cfg}.json")
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        parse(sys.argv[2], sys.argv[3])
