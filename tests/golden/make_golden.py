"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libsogref.so,
built from /root/reference/proj/include by oracle/Makefile).  Run here, where the
reference exists; the fixtures are committed so the GPU box (no /root/reference) can
check the oracle and the host generators against the reference's own outputs.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bindings import BRANCH, CONSTANT, DDA, HDDA, LINEAR, SKIP, RefLib  # noqa: E402

R = RefLib()


def grid_arrays(prefix, g, out):
    out[f"{prefix}_res"] = np.asarray(g.res, np.int32)
    out[f"{prefix}_wmin"] = np.asarray(g.wmin, np.float64)
    out[f"{prefix}_voxel"] = np.float64(g.voxel)
    out[f"{prefix}_bits"] = g.bits


def main():
    out = {}
    # 1) scenes (generate_scene) at 32^3/64^3 and their SOG1 bytes (build_sparse + serialize_sparse)
    scenes = [("blobs", 32, 1, 0.05, 12), ("shell", 48, 1, 0.05, 12), ("sponge", 32, 2, 0.05, 12),
              ("random", 32, 3, 0.1, 12), ("blobs", 40, 4, 0.05, 48)]
    for i, (kind, res, seed, frac, count) in enumerate(scenes):
        g = R.scene(kind, res, seed=seed, fraction=frac, count=count)
        grid_arrays(f"scene{i}", g, out)
        out[f"scene{i}_meta"] = np.array([["blobs", "shell", "sponge", "random"].index(kind), res, seed, count], np.int64)
        out[f"scene{i}_frac"] = np.float64(frac)
        out[f"scene{i}_sog1"] = np.frombuffer(R.sog1(g), np.uint8)
    # odd resolution + multi-region grids (padding, root entries)
    for i, (res, seed, bf, nf) in enumerate([((11, 5, 9), 9, 0.4, 0.05), ((136, 8, 130), 77, 0.05, 0.001)]):
        g = R.random_blocky_grid(res, (-1.0, -1.0, -1.0), 2.0 / res[0], seed, bf, nf)
        grid_arrays(f"blocky{i}", g, out)
        out[f"blocky{i}_args"] = np.array([seed, bf, nf], np.float64)
        out[f"blocky{i}_sog1"] = np.frombuffer(R.sog1(g), np.uint8)
    # 2) rays: random_ray, make_probe_rays, camera
    g0 = R.scene("blobs", 32, seed=1)
    out["rays_random"] = R.random_rays(g0, 200, 7)
    out["rays_probe"] = R.probe_rays(g0, 200, 11)
    out["rays_camera"] = R.camera_rays(width=21, height=15)
    # 3) sampler outputs through sog::run_sampler / run_cascade_sampler (+ recorded cells)
    cases = []
    for si in (0, 2, 3):
        for rays_name in ("rays_random", "rays_camera"):
            for an, k in ((DDA, BRANCH), (DDA, SKIP), (HDDA, BRANCH), (HDDA, SKIP)):
                for sk, dt, gr in ((CONSTANT, 0.5 * 2.0 / out[f"scene{si}_res"][0], 0.0), (LINEAR, 0.011, 1.0 / 128)):
                    cases.append((si, rays_name, an, k, sk, dt, gr))
    for ci, (si, rays_name, an, k, sk, dt, gr) in enumerate(cases):
        from oracle_bindings import Grid

        g = Grid(tuple(out[f"scene{si}_res"]), tuple(out[f"scene{si}_wmin"]), float(out[f"scene{si}_voxel"]),
                 out[f"scene{si}_bits"])
        p = R.sampler([g], an, k, sk, dt, gr).sample(out[rays_name])
        out[f"case{ci}_args"] = np.array([si, ["rays_random", "rays_camera"].index(rays_name), an, k, sk, dt, gr], np.float64)
        for f in ("packed_info", "t_starts", "t_ends", "cells", "levels", "counters"):
            out[f"case{ci}_{f}"] = getattr(p, f)
    out["n_cases"] = np.int64(len(cases))
    # cascade (build_dense_cascade) + random rays over the coarsest level, linear schedule
    lv = R.cascade("blobs", 4, 32, seed=1)
    for b, g in enumerate(lv):
        grid_arrays(f"casc{b}", g, out)
    rays = R.random_rays(lv[-1], 200, 5)
    out["casc_rays"] = rays
    for an, k in ((DDA, BRANCH), (HDDA, SKIP)):
        p = R.sampler(lv, an, k, LINEAR, 0.013, 1.0 / 256).sample(rays)
        for f in ("packed_info", "t_starts", "t_ends", "cells", "levels", "counters"):
            out[f"casc_an{an}k{k}_{f}"] = getattr(p, f)
    # 4) traversal event streams (collect_events) for a handful of rays
    g = Grid(tuple(out["scene0_res"]), tuple(out["scene0_wmin"]), float(out["scene0_voxel"]), out["scene0_bits"])
    for an in (DDA, HDDA):
        s = R.sampler([g], an, SKIP, CONSTANT, 0.03)
        evs, ts, ns = [], [], []
        for r in out["rays_random"][:20]:
            n, ev, ctr = s.events(r)
            ns.append((n, ctr[0], ctr[1]))
            for e in ev:
                evs.append([*e[0], e[1], e[4], e[5]])
                ts.append([e[2], e[3]])
        out[f"events_an{an}_n"] = np.asarray(ns, np.int64)
        out[f"events_an{an}_ev"] = np.asarray(evs, np.int32)
        out[f"events_an{an}_t"] = np.asarray(ts, np.float64)
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    sz = os.path.getsize(os.path.join(HERE, "reference_golden.npz"))
    print(f"wrote reference_golden.npz ({sz} bytes, {len(out)} arrays, {len(cases)} sampler cases)")


if __name__ == "__main__":
    main()
