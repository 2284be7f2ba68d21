"""BASELINE config 5 / SURVEY §8(d) cfg 5: batched throughput sweep on one GPU.

1M-64M probe rays per launch (powers of 2, `make_probe_rays`, bench.hpp:628-649) on
(i) `random_blocky_grid` (test_support.hpp:41-62, block_fraction in {0.005 ... 0.5}, voxel
noise 0.001) and (ii) iid `random` occupancy (scene_gen.hpp:170-186, fraction in
{0.005 ... 0.5}), 128^3, constant dt0 = voxel / 2.  For every grid: the VDB build (K1) time and,
per ray count, one full sample launch (count -> scan -> total read back -> write of
t_starts / t_ends / ray_indices / cells / levels) for sparse+hdda+skip and dense+dda+branch.
Reports rays/s, samples/s, build vs traversal time and the HDDA / DDA ratio vs occupancy
(the crossover).  Launches whose outputs would exceed --out-cap-gb are skipped and reported.

    python tools/sweep_cfg5.py --out gpurun_out/cfg5
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_10272_b200 as P  # noqa: E402

FRACTIONS = [0.005, 0.01, 0.02, 0.05, 0.1, 0.2, 0.5]
BYTES_PER_SAMPLE = 8 + 8 + 4 + 4 + 1  # t_start, t_end, ray_index, cell, level


def timed(fn, reps):
    outs, times = [], []  # outputs kept until the end: no destructor inside a timed region
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        outs.append(fn())
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    timed.last = times
    return sorted(times)[len(times) // 2], outs[-1]


def split_ms(s, r, packed, total, outs):
    """One more launch with events around each pass: (count incl. scan, write) ms."""
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    ev[0].record()
    s.count(r, packed_info=packed)
    ev[1].record()
    s.write(r, packed, total, out=outs)
    ev[2].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--res", type=int, default=128)
    ap.add_argument("--log2-min", type=int, default=20)
    ap.add_argument("--log2-max", type=int, default=26)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out-cap-gb", type=float, default=48.0)
    ap.add_argument("--out", default="gpurun_out/cfg5")
    ap.add_argument("--fractions", default=",".join(str(f) for f in FRACTIONS))
    ap.add_argument("--families", default="blocky,random")
    a = ap.parse_args()
    fracs = [float(x) for x in a.fractions.split(",")]
    fams = a.families.split(",")
    os.makedirs(a.out, exist_ok=True)
    t = P.GridTransform.cube(a.res, (-1.0, -1.0, -1.0), 2.0)
    sched = P.StepSchedule.constant(0.5 * t.voxel_size)
    nmax = 1 << a.log2_max
    rays_h = P.make_probe_rays(t, nmax, 5)
    rays = torch.from_numpy(rays_h).cuda()
    del rays_h
    rows = []
    for family in fams:
        for f in fracs:
            bits = (P.random_blocky_grid(t, 7, f, 0.001) if family == "blocky"
                    else P.random_grid(t, 7, f))
            occ = float(np.unpackbits(bits, bitorder="little")[:t.voxel_count()].mean())
            dense = P.DenseGrid(t, bits)
            build_ms, sparse = timed(lambda: P.build_sparse(dense), 10)
            variants = {"sparse+hdda+skip": P.Sampler([sparse], P.Analyzer.hdda, P.KernelKind.skip, sched),
                        "dense+dda+branch": P.Sampler([dense], P.Analyzer.dda, P.KernelKind.branch, sched)}
            for lg in range(a.log2_min, a.log2_max + 1):
                n = 1 << lg
                r = rays[:n]
                for name, s in variants.items():
                    packed, st = s.count(r)
                    total = int(st.cpu()[P.STAT_TOTAL_SAMPLES])
                    row = {"family": family, "fraction": f, "occupancy": occ, "leaves": sparse.leaf_count(),
                           "vdb_bytes": sparse.memory_bytes(), "build_ms": build_ms, "variant": name,
                           "rays": n, "samples": total}
                    if total * BYTES_PER_SAMPLE > a.out_cap_gb * 1e9:
                        row["status"] = f"skipped: outputs {total * BYTES_PER_SAMPLE / 1e9:.0f} GB > cap"
                        rows.append(row)
                        continue
                    outs = {"t_starts": torch.empty(total, dtype=torch.float64, device="cuda"),
                            "t_ends": torch.empty(total, dtype=torch.float64, device="cuda"),
                            "ray_indices": torch.empty(total, dtype=torch.int32, device="cuda"),
                            "cells": torch.empty(total, dtype=torch.int32, device="cuda"),
                            "levels": torch.empty(total, dtype=torch.uint8, device="cuda")}

                    def launch():  # the whole two-pass launch, total read back in between
                        pk, stt = s.count(r, packed_info=packed)
                        tot = int(stt.cpu()[P.STAT_TOTAL_SAMPLES])
                        s.write(r, pk, tot, out=outs)
                        return tot

                    launch()
                    ms, tot = timed(launch, a.reps)
                    assert tot == total
                    row["rep_ms"] = timed.last
                    row["count_ms"], row["write_ms"] = split_ms(s, r, packed, total, outs)
                    row["free_gb"] = torch.cuda.mem_get_info()[0] / 1e9
                    _, stt = s.count(r, packed_info=packed)
                    row["slab_overflow_rays"] = int(stt.cpu()[P.STAT_SLAB_OVERFLOW_RAYS])
                    row.update(status="ok", ms=ms, rays_per_s=n / ms * 1e3, samples_per_s=total / ms * 1e3,
                               samples_per_ray=total / n, build_over_launch=build_ms / ms)
                    rows.append(row)
                    del outs
                    print(f"{family:6s} f={f:<6} occ={occ:.4f} {name:18s} n=2^{lg} {ms:9.3f} ms "
                          f"{n / ms / 1e3:9.1f} Mrays/s {total / ms / 1e6:8.2f} Gsamples/s  count {row['count_ms']:.2f} "
                          f"write {row['write_ms']:.2f} ms  reps {[round(x, 2) for x in row['rep_ms']]} "
                          f"overflow {row['slab_overflow_rays']} free {row['free_gb']:.0f} GB", flush=True)
            del variants, sparse, dense
            P.release_workspaces()
    json.dump({"config": "cfg5", "res": a.res, "dt0": 0.5 * t.voxel_size, "rows": rows},
              open(os.path.join(a.out, "cfg5_sweep.json"), "w"), indent=1)
    # crossover table: HDDA / DDA rays/s per occupancy at each ray count
    lines = ["family,fraction,occupancy,rays,hdda_Mrays_s,dda_Mrays_s,hdda_over_dda,build_ms,hdda_launch_ms"]
    idx = {(r["family"], r["fraction"], r["rays"], r["variant"]): r for r in rows}
    for family in fams:
        for f in fracs:
            for lg in range(a.log2_min, a.log2_max + 1):
                h = idx.get((family, f, 1 << lg, "sparse+hdda+skip"))
                d = idx.get((family, f, 1 << lg, "dense+dda+branch"))
                if not h or not d or h["status"] != "ok" or d["status"] != "ok":
                    continue
                lines.append(f"{family},{f},{h['occupancy']:.4f},{1 << lg},{h['rays_per_s'] / 1e6:.1f},"
                             f"{d['rays_per_s'] / 1e6:.1f},{h['rays_per_s'] / d['rays_per_s']:.2f},"
                             f"{h['build_ms']:.3f},{h['ms']:.3f}")
    open(os.path.join(a.out, "cfg5_crossover.csv"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
