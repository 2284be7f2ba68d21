#!/usr/bin/env python3
"""bench.py — rays/s and samples/s of the B200 VDB+HDDA sampler (arXiv 2404.10272 hot path).

Default workload = BASELINE.json configs[1], "NeRF-Synthetic-shaped sweep": 8 procedural
128^3 object grids of varying sparsity (SURVEY §8d cfg 2), 200 views of 800x800 each on
an orbit through the bench camera pose (1.9, 1.4, 2.3) -> 0, vfov 42 deg.  One step = one
view of each of the 8 objects (8 x 640,000 rays), sharded over ranks by view (weak
scaling: every rank does one view per object per step).  Per object and step the product
path runs pass 1 (count + fused scan) and pass 2 (write) of `sparse+hdda+skip` through the
C-ABI; the paper's dense baseline `dense+dda+branch` (and its skip twin) is timed the same
way.  Rays are materialized in HBM before the timed region (distinct per object and step:
328 MB of rays + ~1-2 GB of samples per step > the 126 MB L2, so no explicit L2 flush).

JSON line keys follow the driver contract; see DESIGN.md §Measurement for the roofline basis.
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2|cfg1|cfg3|cfg4]
  python bench.py --impl reference ...   (the reference CPU sampler on the host cores)
"""
from __future__ import annotations

import argparse
from concurrent.futures import ThreadPoolExecutor
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(1, os.path.join(ROOT, "tests"))  # oracle_bindings: CPU-baseline leg only

from paper_2404_10272_b200.shard import broadcast_payload, view_of  # noqa: E402

CAM_POS = (1.9, 1.4, 2.3)
N_VIEWS = 200

# cfg 2: 8 procedural 128^3 objects of varying sparsity
CFG2_OBJECTS = [
    ("shell", dict(seed=1, count=12)),
    ("shell", dict(seed=2, count=256)),
    ("blobs", dict(seed=1, count=6)),
    ("blobs", dict(seed=2, count=12)),
    ("blobs", dict(seed=3, count=24)),
    ("blobs", dict(seed=4, count=48)),
    ("sponge", dict(seed=1)),
    ("random", dict(seed=1, fraction=0.02)),
]


def orbit_camera(P, view: int, width=800, height=800):
    """View v of the orbit: the bench pose rotated about +y by 2*pi*v/200 (v = 0 is cfg 1)."""
    th = 2.0 * math.pi * (view % N_VIEWS) / N_VIEWS
    x, y, z = CAM_POS
    pos = (x * math.cos(th) + z * math.sin(th), y, -x * math.sin(th) + z * math.cos(th))
    return P.Camera(pos, (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, width, height)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every 5 ms while the timed region runs
    (nvidia-smi's own polling starts too slowly for a sub-second region); falls back to
    `nvidia-smi -lms` when NVML is unavailable."""

    # nvmlClocksEventReasons bits (nvml.h)
    BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index, self.rows, self.stop = index, [], threading.Event()
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            get_r = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons

            def poll():
                while not self.stop.is_set():
                    try:
                        self.rows.append((float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)), int(get_r(h))))
                    except Exception:
                        pass
                    time.sleep(0.005)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t is not None:
            self.t.join(timeout=1)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for _, m in self.rows for b, name in self.BITS.items() if m & b})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml"}


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
class Workload:
    """Grids (per object) + a ray generator per (step, object) + the schedule."""

    def __init__(self, P, name: str):
        self.P, self.name = P, name
        self.ray_order = 0
        base = P.GridTransform.cube(128, (-1.0, -1.0, -1.0), 2.0)
        self.cascade = False
        self.schedule = P.StepSchedule.constant(0.5 * base.voxel_size)
        if name == "cfg2":
            self.objects = []
            for kind, kw in CFG2_OBJECTS:
                bits, occ = P.generate_scene(kind, base, **kw)
                self.objects.append(dict(label=f"{kind}:{kw}", levels=[(base, bits)], occupancy=occ,
                                         scene=(kind, kw.get("seed", 1), kw.get("count", 12), base)))
            self.width = self.height = 800
            self.desc = ("8 procedural 128^3 objects (shell s1, shell s2 n256, blobs s1..s4 n6..48, "
                         "sponge s1, random 2%), 800x800 orbit views, dt0 = half voxel")
        elif name == "cfg1":
            bits, occ = P.generate_scene("shell", base, seed=1)
            self.objects = [dict(label="shell s1", levels=[(base, bits)], occupancy=occ,
                                 scene=("shell", 1, 12, base))]
            self.width = self.height = 800
            self.desc = "single-level 128^3 shell s1, 800x800 bench camera, dt0 = half voxel"
        elif name == "cfg3":
            lv = P.build_dense_cascade("blobs", base, 4, seed=1)
            self.objects = [dict(label="blobs s1 x4 cascade", levels=lv, occupancy=None,
                                 scene=("blobs", 1, 12, base))]
            self.cascade = True
            self.width, self.height = 1297, 840
            self.schedule = P.StepSchedule.linear(0.5 * base.voxel_size, 1.0 / 256.0)
            self.desc = "4-level 128^3 blobs s1 cascade, 1297x840 bench camera, linear dt0=2^-7 growth 1/256"
        elif name == "cfg4":
            t512 = P.GridTransform.cube(512, (-1.0, -1.0, -1.0), 2.0)
            bits, occ = P.generate_scene("blobs", t512, seed=1)
            self.objects = [dict(label="blobs s1 512^3", levels=[(t512, bits)], occupancy=occ)]
            self.schedule = P.StepSchedule.constant(0.5 * t512.voxel_size)
            self.n_probe = 1 << 24
            self.ray_order = 1  # incoherent probe rays: pass 1 bins them (sogk_sampler_set_ray_order)
            self.desc = ("512^3 blobs s1 (1.44%), 2^24 make_probe_rays, dt0 = half voxel; pass 1 "
                         "processes the rays binned by grid entry cell and direction")
        else:
            raise SystemExit(f"unknown config {name}")

    def camera(self, step_index: int, obj: int, rank: int, world: int):
        """The camera of (global step, object) for this rank (None for probe-ray configs)."""
        if self.name == "cfg4":
            return None
        view = view_of(step_index, rank, world, N_VIEWS, obj * (N_VIEWS // max(1, len(self.objects))))
        if self.name in ("cfg1", "cfg3"):
            view = 0
        return orbit_camera(self.P, view, self.width, self.height)

    def rays_per_object(self) -> int:
        return self.n_probe if self.name == "cfg4" else self.width * self.height

    def fill_rays(self, out, step_index: int, obj: int, rank: int, world: int):
        """Write the rays of (global step, object) for this rank into the CUDA tensor `out`."""
        P = self.P
        if self.name == "cfg4":
            import torch

            t = self.objects[0]["levels"][0][0]
            h = P.make_probe_rays(t, self.n_probe, seed=1000 + step_index * world + rank)
            out.copy_(torch.from_numpy(h))
            return
        view = view_of(step_index, rank, world, N_VIEWS, obj * (N_VIEWS // max(1, len(self.objects))))
        if self.name in ("cfg1", "cfg3"):
            view = 0  # the bench camera pose of the config
        cam = orbit_camera(P, view, self.width, self.height)
        cam.rays_device(0, self.width * self.height, out=out)

    def host_rays(self, step_index: int, obj: int, rank: int, world: int) -> np.ndarray:
        P = self.P
        if self.name == "cfg4":
            t = self.objects[0]["levels"][0][0]
            return P.make_probe_rays(t, self.n_probe, seed=1000 + step_index * world + rank)
        view = view_of(step_index, rank, world, N_VIEWS, obj * (N_VIEWS // max(1, len(self.objects))))
        if self.name in ("cfg1", "cfg3"):
            view = 0  # the bench camera pose of the config
        return orbit_camera(P, view, self.width, self.height).rays()


def grid_bytes(P, levels_bits, analyzer):
    if analyzer == P.Analyzer.dda:
        return sum(int(b.size) for _, b in levels_bits)
    return None  # filled from the VDB info


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2404_10272_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    wl = Workload(P, args.config)
    n_obj = len(wl.objects)
    # --- grids: rank 0's payloads broadcast once over NVLink (NCCL), VDB built per rank (K1)
    grids = []
    build_ms = []
    dist_ms = []
    dist_grids = []
    for o in wl.objects:
        dense_lv, vdb_lv, cd_lv = [], [], []
        for t, bits in o["levels"]:
            d_bits = torch.from_numpy(bits).to(dev)
            broadcast_payload(d_bits)  # once, NCCL over NVLink; rank 0's payload wins
            dg = P.DenseGrid(t, d_bits)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            vg = P.build_sparse(dg)
            e1.record()
            torch.cuda.synchronize()
            build_ms.append(e0.elapsed_time(e1))
            e0.record()
            cg = P.build_distance(dg)
            e1.record()
            torch.cuda.synchronize()
            dist_ms.append(e0.elapsed_time(e1))
            dense_lv.append(dg)
            vdb_lv.append(vg)
            cd_lv.append(cg)
        grids.append((dense_lv, vdb_lv))
        dist_grids.append(cd_lv)
    vdb_bytes = [sum(int(v.memory_bytes()) for v in vl) for _, vl in grids]
    dense_bytes = [sum(int(t.payload_bytes()) for t, _ in o["levels"]) for o in wl.objects]

    variants = {
        "hdda_skip": (P.Analyzer.hdda, P.KernelKind.skip),
        "dda_branch": (P.Analyzer.dda, P.KernelKind.branch),
        "dda_skip": (P.Analyzer.dda, P.KernelKind.skip),
        "cd_skip": (P.Analyzer.cd, P.KernelKind.skip),
    }
    if args.variants:
        variants = {k: v for k, v in variants.items() if k in args.variants.split(",")}
    samplers = {}
    for vname, (an, kk) in variants.items():
        samplers[vname] = [P.Sampler(grids[i][1] if an == P.Analyzer.hdda else
                                     dist_grids[i] if an == P.Analyzer.cd else grids[i][0], an, kk,
                                     wl.schedule, cascade=wl.cascade, ray_order=wl.ray_order)
                           for i in range(n_obj)]

    nr = wl.rays_per_object()
    steps_total = args.warmup + args.steps
    # --- rays for every (step, object) in HBM before timing
    rays = [[torch.empty((nr, 8), dtype=torch.float64, device=dev) for _ in range(n_obj)]
            for _ in range(steps_total)]
    for s in range(steps_total):
        for o in range(n_obj):
            wl.fill_rays(rays[s][o], s, o, rank, world)
    torch.cuda.synchronize()

    # parts: the units one count/write pair processes -- one per object, or, for single-object
    # configs on several streams, one contiguous ray range per stream (each its own packed batch)
    if n_obj == 1 and args.streams > 1:
        cut = [nr * i // args.streams for i in range(args.streams + 1)]
        parts = [(0, cut[i], cut[i + 1]) for i in range(args.streams)]
    else:
        parts = [(o, 0, nr) for o in range(n_obj)]
    n_parts = len(parts)

    def prays(s_, pi):
        o, a, b = parts[pi]
        return rays[s_][o][a:b]

    packed = [torch.empty((b - a, 2), dtype=torch.int64, device=dev) for _, a, b in parts]
    stats = [torch.zeros(8, dtype=torch.int64, device=dev) for _ in parts]
    # --- sizing pass (untimed): totals of every (step, part) -> output capacity per part
    totals = {}
    cap = [0] * n_parts
    for vname, smp in samplers.items():
        for s in range(steps_total):
            for pi, (o, a, b) in enumerate(parts):
                smp[o].count(prays(s, pi), packed_info=packed[pi], stats=stats[pi])
                tot = int(stats[pi][0].item())
                totals[(vname, s, pi)] = tot
                cap[pi] = max(cap[pi], tot)
    outs = []
    for pi in range(n_parts):
        c = max(1, cap[pi])
        outs.append(dict(t_starts=torch.empty(c, dtype=torch.float64, device=dev),
                         t_ends=torch.empty(c, dtype=torch.float64, device=dev),
                         ray_indices=torch.empty(c, dtype=torch.int32, device=dev),
                         cells=torch.empty(c, dtype=torch.int32, device=dev)))
    # object totals (the e2e leg's capacities)
    obj_cap = [0] * n_obj
    for vname in samplers:
        for s in range(steps_total):
            per = [0] * n_obj
            for pi, (o, a, b) in enumerate(parts):
                per[o] += totals[(vname, s, pi)]
            for o in range(n_obj):
                obj_cap[o] = max(obj_cap[o], per[o])
    # hit rays per (step, part) for the write kernel's algorithmic bytes
    hits = {}
    for s in range(steps_total):
        for pi, (o, a, b) in enumerate(parts):
            smp = samplers[next(iter(samplers))][o]
            smp.count(prays(s, pi), packed_info=packed[pi], stats=stats[pi])
            hits[(s, pi)] = int((packed[pi][:, 1] > 0).sum().item())

    stream = torch.cuda.current_stream()
    results = {}
    for vname, smp in samplers.items():
        def one_step(s, ev=None):
            for pi, (o, a, b) in enumerate(parts):
                if ev is not None:
                    ev[pi][0].record(stream)
                smp[o].count(prays(s, pi), packed_info=packed[pi], stats=stats[pi])
                if ev is not None:
                    ev[pi][1].record(stream)
                smp[o].write(prays(s, pi), packed[pi], totals[(vname, s, pi)], ray_index_base=a,
                             out=outs[pi], cells=True, levels=False)
                if ev is not None:
                    ev[pi][2].record(stream)

        for s in range(args.warmup):
            one_step(s)
        evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_parts)]
               for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            t0.record(stream)
            for k in range(args.steps):
                one_step(args.warmup + k, evs[k])
            t1.record(stream)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = t0.elapsed_time(t1)
        ms_serial = ms
        if args.streams > 1:
            # the same steps with objects spread over `streams` CUDA streams (each stream has
            # its own pass-1 -> pass-2 workspace): one object's pass 2 (memory-bound) overlaps
            # the next object's pass 1 (issue-bound); sizes are precomputed, no host sync
            side = [torch.cuda.Stream(device=dev) for _ in range(args.streams)]

            def step_overlapped(s):
                for pi, (o, a, b) in enumerate(parts):
                    st = side[pi % args.streams]
                    smp[o].count(prays(s, pi), packed_info=packed[pi], stats=stats[pi], stream=st)
                    smp[o].write(prays(s, pi), packed[pi], totals[(vname, s, pi)], ray_index_base=a,
                                 out=outs[pi], cells=True, levels=False, stream=st)

            for st in side:
                st.wait_stream(stream)
            for s in range(args.warmup):
                step_overlapped(s)
            for st in side:
                stream.wait_stream(st)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            u0 = torch.cuda.Event(enable_timing=True)
            u1 = torch.cuda.Event(enable_timing=True)
            with ClockSampler(local) as clk:
                u0.record(stream)
                for st in side:
                    st.wait_event(u0)
                for k in range(args.steps):
                    step_overlapped(args.warmup + k)
                for st in side:
                    stream.wait_stream(st)
                u1.record(stream)
                torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            ms = u0.elapsed_time(u1)
        count_ms = sum(evs[k][pi][0].elapsed_time(evs[k][pi][1]) for k in range(args.steps) for pi in range(n_parts))
        write_ms = sum(evs[k][pi][1].elapsed_time(evs[k][pi][2]) for k in range(args.steps) for pi in range(n_parts))
        samples = sum(totals[(vname, args.warmup + k, pi)] for k in range(args.steps) for pi in range(n_parts))
        nhit = sum(hits[(args.warmup + k, pi)] for k in range(args.steps) for pi in range(n_parts))
        results[vname] = dict(ms=ms, ms_serial=ms_serial, count_ms=count_ms, write_ms=write_ms, samples=samples,
                              hit_rays=nhit, clocks=clk.summary())

    P.release_workspaces()
    # --- render leg: render_frame fused (sample + composite per pixel, no sample arrays),
    # the paper's rendered-frames metric; one frame = one object's view
    render = None
    if not args.no_render and wl.name != "cfg4":
        scenes = [P.analytic_scene(o["scene"][0], o["scene"][3], seed=o["scene"][1], count=o["scene"][2])
                  for o in wl.objects]
        npx = wl.width * wl.height
        r_res = torch.empty((npx, 5), dtype=torch.float64, device=dev)
        r_rgb = torch.empty((npx, 3), dtype=torch.uint8, device=dev)
        r_st = torch.zeros(8, dtype=torch.int64, device=dev)
        render = {}
        for vname, smp in samplers.items():
            def rstep(s_):
                for o in range(n_obj):
                    cam = wl.camera(s_, o, rank, world)._c()
                    P._check(P.lib.sogk_render_camera(smp[o]._h, scenes[o].handle, P.C.byref(cam), 0, npx,
                                                      r_res.data_ptr(), r_rgb.data_ptr(), r_st.data_ptr(),
                                                      stream.cuda_stream or None), "render")
            for s_ in range(args.warmup):
                rstep(s_)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for k in range(args.steps):
                rstep(args.warmup + k)
            e1.record(stream)
            torch.cuda.synchronize()
            rms = e0.elapsed_time(e1)
            frames = args.steps * n_obj
            render[vname] = {"frames_per_sec": frames / (rms / 1e3), "ms_per_frame": rms / frames,
                             "mpix_per_sec": frames * npx / (rms / 1e3) / 1e6}

    # --- e2e through the host C-ABI entry point (pinned host buffers, H2D/D2H timed)
    e2e = None
    P.release_workspaces()  # the timing legs' per-stream workspaces
    if not args.no_e2e:
        smp = samplers[next(iter(samplers))]
        vname0 = next(iter(samplers))
        h_rays = []
        for s in range(steps_total):
            row = []
            for o in range(n_obj):
                t = torch.empty((nr, 8), dtype=torch.float64, pin_memory=True)
                t.copy_(rays[s][o], non_blocking=False)
                row.append(t)
            h_rays.append(row)
        hcap = max(obj_cap)
        n_workers = max(1, min(args.e2e_workers, n_obj))

        def host_outputs():  # pinned output buffers, one set per worker thread
            o = dict(packed_info=torch.empty((nr, 2), dtype=torch.int64, pin_memory=True).numpy(),
                     t_starts=torch.empty(hcap, dtype=torch.float64, pin_memory=True).numpy(),
                     t_ends=torch.empty(hcap, dtype=torch.float64, pin_memory=True).numpy(),
                     ray_indices=torch.empty(hcap, dtype=torch.int32, pin_memory=True).numpy(),
                     cells=torch.empty(hcap, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32),
                     stats=np.zeros(8, np.int64))
            o["counters"] = torch.empty((nr, 3), dtype=torch.int32, pin_memory=True).numpy()
            return o

        h_outs = [host_outputs() for _ in range(n_workers)]
        lib = P.lib
        pool = ThreadPoolExecutor(n_workers) if n_workers > 1 else None

        def e2e_objects(s, full, w):
            # full: the packed intervals (t_starts, t_ends, ray_indices, cells); otherwise what
            # the reference's run_sampler returns per ray (sampling.hpp:157-164): its sample
            # buffer (packed t_starts + packed_info) and its three counters.  Worker w takes the
            # objects o = w mod n_workers (independent samplers: each call is synchronous and
            # pipelines its own chunks; ctypes drops the GIL, so the calls overlap)
            h_out = h_outs[w]
            for o in range(w, n_obj, n_workers):
                rc = lib.sogk_sample_host(smp[o]._h, h_rays[s][o].data_ptr(), nr, 0, hcap,
                                          h_out["packed_info"].ctypes.data, h_out["t_starts"].ctypes.data,
                                          h_out["t_ends"].ctypes.data if full else None,
                                          h_out["ray_indices"].ctypes.data if full else None,
                                          h_out["cells"].ctypes.data if full else None, None, None,
                                          None if full else h_out["counters"].ctypes.data,
                                          h_out["stats"].ctypes.data, stream.cuda_stream or None)
                P._check(rc, "sample_host")

        def e2e_step(s, full):
            if pool is None:
                e2e_objects(s, full, 0)
            else:
                for f in [pool.submit(e2e_objects, s, full, w) for w in range(n_workers)]:
                    f.result()

        def timed(full):
            for s in range(args.warmup):
                e2e_step(s, full)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ts = time.perf_counter()
            for k in range(args.steps):
                e2e_step(args.warmup + k, full)
            torch.cuda.synchronize()
            sec = time.perf_counter() - ts
            if world > 1:
                tt = torch.tensor([sec], device=dev, dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                sec = float(tt.item())
            return sec

        e2e_s = timed(False)
        e2e_full_s = timed(True)
        samples0 = sum(totals[(vname0, args.warmup + k, pi)] for k in range(args.steps) for pi in range(n_parts))
        if pool is not None:
            pool.shutdown()
        e2e = dict(seconds=e2e_s, h2d=nr * 64 * n_obj, workers=n_workers,
                   d2h_per_run=samples0 * 8 / args.steps + nr * (16 + 12) * n_obj,
                   full_seconds=e2e_full_s, full_d2h=samples0 * 24 / args.steps + nr * 16 * n_obj)

    # --- max over ranks
    def rmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def rsum(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    agg = {}
    for vname, r in results.items():
        agg[vname] = dict(ms=rmax(r["ms"]), ms_serial=rmax(r["ms_serial"]), samples=rsum(r["samples"]),
                          count_ms=r["count_ms"],
                          write_ms=r["write_ms"], hit_rays=r["hit_rays"], local_samples=r["samples"],
                          clocks=r["clocks"])
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    head = "hdda_skip" if "hdda_skip" in agg else next(iter(agg))
    h = agg[head]
    total_rays = nr * n_obj * args.steps * world
    sec = h["ms"] / 1e3
    rays_s = total_rays / sec
    samples_s = h["samples"] / sec
    peak, peak_src = load_peaks()
    # roofline: dominant kernel (larger share of the step) with its algorithmic bytes
    # (SURVEY §8(d)): pass 1 reads the rays (64 B) and writes packed_info (16 B) per ray;
    # pass 2 reads packed_info (16 B/ray) and writes the samples (24 B each).  The slabs
    # pass 1 hands to pass 2 (12 B/sample each way) are not algorithmic; ncu's DRAM bytes
    # (`traffic`, profiles/traffic_<cfg>.json) show them.
    launches = args.steps * n_parts
    nr_loc = nr * n_obj * args.steps
    write_bytes = nr_loc * 16 + h["local_samples"] * 24
    count_bytes = nr_loc * (64 + 16)
    pass2 = {"kernel": "gather_kernel + tail_kernel (pass 2)", "ms": h["write_ms"], "bytes": write_bytes}
    pass1 = {"kernel": "count_kernel + scan_kernel (pass 1)", "ms": h["count_ms"], "bytes": count_bytes}
    dom, other = (pass2, pass1) if h["write_ms"] >= h["count_ms"] else (pass1, pass2)

    def gbs(k):
        return k["bytes"] / launches / (k["ms"] / launches / 1e3) / 1e9

    achieved = gbs(dom)
    step_bytes = nr_loc * (64 + 16) + h["local_samples"] * 24 + sum(vdb_bytes) * args.steps
    step_gbs = step_bytes / (h["ms"] / 1e3) / 1e9
    traffic = {}
    tf = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf))
        except Exception:
            traffic = {}
    # the capture's launch covered `rays_per_launch` rays: scale to this run's launches
    rays_per_launch_here = nr_loc / launches
    tscale = rays_per_launch_here / traffic.get("rays_per_launch", rays_per_launch_here)
    for key in ("pass1", "pass2"):
        if key in traffic and traffic[key].get("dram_bytes_per_launch"):
            traffic[key]["dram_bytes_per_launch"] = traffic[key]["dram_bytes_per_launch"] * tscale
    dom_key = "pass1" if dom is pass1 else "pass2"
    other_key = "pass2" if dom is pass1 else "pass1"
    # pass 1's real ceiling is instruction issue: warp instructions of one step's
    # count_kernel launches (ncu, profiles/issue_<cfg>.json, tools/issue_probe.py) over the live
    # pass-1 time, against 4 issue slots per SM per clock at the clock measured under load
    issue = None
    isf = os.path.join(ROOT, "profiles", f"issue_{args.config}.json")
    if os.path.exists(isf) and head == "hdda_skip" and world == 1:
        try:
            ij = json.load(open(isf))
            sm_mhz = (h["clocks"] or {}).get("sm_mhz") or 0
            n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
            ipeak = n_sm * 4 * sm_mhz * 1e6
            iach = ij["pass1_warp_inst_per_step"] / (h["count_ms"] / args.steps / 1e3)
            issue = {"bound": "issue", "kernel": "count_kernel (pass 1; time incl. scan_kernel)",
                     "achieved": iach, "peak": ipeak, "unit": "warp-inst/s",
                     "frac": iach / ipeak if ipeak else None,
                     "warp_inst_per_step": ij["pass1_warp_inst_per_step"],
                     "peak_basis": f"{n_sm} SMs x 4 schedulers x {sm_mhz} MHz (median SM clock under load)",
                     "source": ij.get("source")}
        except Exception as e:  # noqa: BLE001
            issue = {"error": str(e)}

    line = {
        "metric": "rays/sec and samples/sec per B200 (and 8-GPU box), HDDA-VDB vs dense-DDA, % HBM roofline",
        "value": rays_s,
        "unit": "rays/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": h["ms"] / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (procedural occupancy grids from the reference generators, camera/probe rays)",
        "config": {"workload": args.config, "desc": wl.desc, "variant": "sparse+hdda+skip" if head == "hdda_skip" else head,
                   "rays_per_step": nr * n_obj * world, "objects": [o["label"] for o in wl.objects],
                   "parallelism": f"rays sharded by view over {world} GPU(s), objects over {args.streams} stream(s)",
                   "l2": "inputs+outputs per step > 126 MB L2 (no flush)"},
        "samples_per_sec": samples_s,
        "samples_per_step": h["samples"] / args.steps,
        "variants": {k: {"rays_per_sec": total_rays / (v["ms"] / 1e3),
                         "samples_per_sec": v["samples"] / (v["ms"] / 1e3),
                         "ms_per_step": v["ms"] / args.steps,
                         "ms_per_step_one_stream": v["ms_serial"] / args.steps,
                         "count_ms_per_step": v["count_ms"] / args.steps,
                         "write_ms_per_step": v["write_ms"] / args.steps} for k, v in agg.items()},
        "hdda_vs_dda_branch": (agg["dda_branch"]["ms"] / agg["hdda_skip"]["ms"]) if {"dda_branch", "hdda_skip"} <= agg.keys() else None,
        "roofline": {"bound": "hbm", "kernel": dom["kernel"], "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic.get(dom_key, {}).get("dram_bytes_per_launch"),
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": dom["bytes"] / launches,
                     "note": "pass 1 is bound by traversal issue/latency and L1/L2 store transactions, "
                             "not HBM (DESIGN.md §4); traffic = ncu dram read+write of one launch "
                             "(object 0), " + traffic.get("source", "no capture committed"),
                     "other_pass": {"kernel": other["kernel"], "achieved": gbs(other), "frac": gbs(other) / peak,
                                    "algorithmic_bytes_per_launch": other["bytes"] / launches,
                                    "traffic": traffic.get(other_key, {}).get("dram_bytes_per_launch")},
                     "issue_ceiling": issue},
        "step_roofline": {"bytes_per_step": step_bytes / args.steps, "achieved_gbs": step_gbs,
                          "frac": step_gbs / peak,
                          "basis": "N_rays*(64+16) + N_samples*24 + VDB bytes (SURVEY §8d)"},
        "vdb_build_ms": build_ms,
        "distance_build_ms": dist_ms,
        "grid_bytes": {"dense": dense_bytes, "vdb_sog1": vdb_bytes},
        "render": ({"what": "render_frame fused on the GPU (Camera::pixel_ray -> sampling -> "
                             "composite_detailed -> Image::set_pixel per pixel, no sample arrays), "
                             f"{wl.width}x{wl.height} frames, rank 0",
                     "variants": render} if render else None),
        "gpu_launches": 4 * launches,  # count, scan, gather, tail per object
        "clocks": h["clocks"],
    }
    if e2e:
        line["e2e"] = {"value": total_rays / e2e["seconds"], "unit": "rays/s",
                       "h2d_bytes_per_step": int(e2e["h2d"]), "d2h_bytes_per_step": int(e2e["d2h_per_run"]),
                       "api": "sogk_sample_host: pinned host rays in; out, what run_sampler returns per ray "
                              "(sampling.hpp:157-164): its samples (packed t_starts + packed_info) and "
                              "its three counters",
                       "host_threads": e2e["workers"],
                       "full_intervals": {"value": total_rays / e2e["full_seconds"], "unit": "rays/s",
                                          "d2h_bytes_per_step": int(e2e["full_d2h"]),
                                          "outputs": "packed_info, t_starts, t_ends, ray_indices, cells"}}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(P, wl, args)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref: the unmodified reference headers) — baseline only
# ---------------------------------------------------------------------------
def _ref_sampler(wl, analyzer, kernel):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bindings import Grid, RefLib

    R = RefLib()
    out = []
    for o in wl.objects:
        lv = [Grid(t.resolution, t.world_min, t.voxel_size, b) for t, b in o["levels"]]
        out.append(R.sampler(lv, analyzer, kernel, wl.schedule.kind, wl.schedule.dt0,
                             wl.schedule.growth, cascade=wl.cascade))
    return R, out


def _cpu_sample(wl, stride, step_index, rank=0, world=1):
    return [wl.host_rays(step_index, o, rank, world)[::stride].copy() for o in range(len(wl.objects))]


def _spin_mask(wl, rays_per_obj):
    """Rays on which the reference HDDA never returns are screened out with the
    capped oracle detector; they are excluded from the CPU timing and counted."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bindings import HDDA, SKIP, Grid, Oracle

    O = Oracle()
    masks = []
    for o, r in zip(wl.objects, rays_per_obj):
        lv = [Grid(t.resolution, t.world_min, t.voxel_size, b) for t, b in o["levels"]]
        s = O.sampler(lv, HDDA, SKIP, wl.schedule.kind, wl.schedule.dt0, wl.schedule.growth,
                      cascade=wl.cascade)
        masks.append((O.sample(s, r).status == 2).astype(np.uint8))
    return masks


def cpu_baseline(P, wl, args):
    from oracle_bindings import HDDA, SKIP

    try:
        R, smp = _ref_sampler(wl, HDDA, SKIP)
    except FileNotFoundError:
        return {"value": None, "unit": "rays/s", "kind": "reference", "cores": 0,
                "sample": "oracle/_ref missing"}
    cores = os.cpu_count() or 1
    stride = args.cpu_stride
    rays = _cpu_sample(wl, stride, 0)
    masks = _spin_mask(wl, rays)
    sec, n = 0.0, 0
    for s, r, m in zip(smp, rays, masks):
        dt, _ = s.time(r, skip=m, threads=cores, reps=1)
        sec += dt
        n += int(r.shape[0] - m.sum())
    return {"value": n / sec, "unit": "rays/s", "cores": cores, "kind": "reference",
            "sample": f"sparse+hdda+skip via sog::run_sampler, every {stride}th ray of step 0 "
                      f"({n} rays over {len(rays)} object(s)), {cores} threads, spin-screened "
                      f"{int(sum(m.sum() for m in masks))} rays"}


def run_reference(args):
    """--impl reference: the reference CPU sampler (oracle/_ref) on the host cores."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2404_10272_b200 as P
    from oracle_bindings import HDDA, SKIP

    wl = Workload(P, args.config)
    try:
        R, smp = _ref_sampler(wl, HDDA, SKIP)
    except FileNotFoundError as e:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not built: {e}"}))
        return
    cores = os.cpu_count() or 1
    stride = args.cpu_stride
    step_rays, step_masks = [], []
    for s in range(args.warmup + args.steps):
        r = _cpu_sample(wl, stride, s, 0, 1)
        step_rays.append(r)
        step_masks.append(_spin_mask(wl, r))
    per_step_rays = [sum(int(x.shape[0] - m.sum()) for x, m in zip(r, mm)) for r, mm in zip(step_rays, step_masks)]

    def step(s):
        t = 0.0
        for sm, r, m in zip(smp, step_rays[s], step_masks[s]):
            dt, _ = sm.time(r, skip=m, threads=cores, reps=1)
            t += dt
        return t

    for s in range(args.warmup):
        step(s)
    total_s = 0.0
    n = 0
    for k in range(args.steps):
        total_s += step(args.warmup + k)
        n += per_step_rays[args.warmup + k]
    v = n / total_s
    line = {
        "impl": "reference",
        "metric": "rays/sec and samples/sec per B200 (and 8-GPU box), HDDA-VDB vs dense-DDA, % HBM roofline",
        "value": v, "unit": "rays/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_s / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "desc": wl.desc, "variant": "sparse+hdda+skip"},
        "cpu_baseline": {"value": v, "unit": "rays/s", "cores": cores, "kind": "reference",
                         "sample": f"every {stride}th ray of each step's views, sog::run_sampler on {cores} threads"},
        "e2e": {"value": v, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default per config, a timed region of >= ~150 ms: cfg1/cfg3 200, cfg2 50, cfg4 10)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4"])
    ap.add_argument("--variants", default="")
    ap.add_argument("--cpu-stride", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-workers", type=int, default=2,
                    help="host threads issuing sogk_sample_host calls for different objects concurrently")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    ap.add_argument("--streams", type=int, default=2,
                    help="CUDA streams the step's objects are spread over (1: one stream)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = {"cfg1": 200, "cfg2": 50, "cfg3": 200, "cfg4": 10}[args.config]
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
