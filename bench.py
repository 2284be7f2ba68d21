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



def _load_shard():
    """paper_2404_10272_b200/shard.py loaded by path: importing it as a submodule would run the
    package __init__ and load libsogk.so, which the reference arm must not do."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "_sogk_shard", os.path.join(ROOT, "paper_2404_10272_b200", "shard.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


_shard = _load_shard()
broadcast_payload, shard_range, view_of = _shard.broadcast_payload, _shard.shard_range, _shard.view_of

CAM_POS = (1.9, 1.4, 2.3)
N_VIEWS = 200
METRIC = "rays/sec and samples/sec per B200 (and 8-GPU box), HDDA-VDB vs dense-DDA, % HBM roofline"

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
DESC = {
    "cfg1": "single-level 128^3 shell s1, 800x800 bench camera, dt0 = half voxel",
    "cfg2": ("8 procedural 128^3 objects (shell s1, shell s2 n256, blobs s1..s4 n6..48, sponge s1, "
             "random 2%), 800x800 orbit views, dt0 = half voxel"),
    "cfg3": "4-level 128^3 blobs s1 cascade, 1297x840 bench camera, linear dt0=2^-7 growth 1/256",
    "cfg4": ("512^3 blobs s1 (1.44%), 2^24 make_probe_rays, dt0 = half voxel; pass 1 processes the "
             "rays binned by grid entry cell and direction"),
}


def orbit_pos(view: int):
    """View v of the orbit: the bench pose rotated about +y by 2*pi*v/200 (v = 0 is cfg 1)."""
    th = 2.0 * math.pi * (view % N_VIEWS) / N_VIEWS
    x, y, z = CAM_POS
    return (x * math.cos(th) + z * math.sin(th), y, -x * math.sin(th) + z * math.cos(th))


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


def workload_config(name: str, world: int, streams: int) -> dict:
    """The bench line's `config`, identical in both arms (it depends on the arguments only)."""
    if name == "cfg2":
        objects = [f"{k}:{kw}" for k, kw in CFG2_OBJECTS]
        rays = 800 * 800 * len(objects) * world
        par = (f"weak: each of {world} GPU(s) samples its own orbit view of every object per step "
               f"(views interleaved over ranks), objects over {streams} CUDA stream(s)")
    else:
        objects = {"cfg1": ["shell s1"], "cfg3": ["blobs s1 x4 cascade"], "cfg4": ["blobs s1 512^3"]}[name]
        rays = {"cfg1": 800 * 800, "cfg3": 1297 * 840, "cfg4": 1 << 24}[name]
        par = (f"strong: the step's rays split into {world} contiguous range(s) of ceil(N/{world}) "
               f"(global ray_indices), ranges over {streams} CUDA stream(s)")
    return {"workload": name, "desc": DESC[name], "variant": "sparse+hdda+skip", "rays_per_step": rays,
            "objects": objects, "parallelism": par,
            "l2": "inputs+outputs per step > 126 MB L2 (no flush)"}


def scaling_of(name: str) -> str:
    return "weak" if name == "cfg2" else "strong"


class ProductGen:
    """Input generation through the package's host generators (libsogk.so; pinned to the
    reference generators by tests/test_host.py) -- the GPU arm."""

    def __init__(self, P):
        self.P = P

    def scene(self, kind, res, seed=1, count=12, fraction=0.05):
        t = self.P.GridTransform.cube(res, (-1.0, -1.0, -1.0), 2.0)
        bits, occ = self.P.generate_scene(kind, t, seed=seed, count=count, fraction=fraction)
        return [(t.resolution, t.world_min, t.voxel_size, bits)], occ

    def cascade(self, kind, res, levels, seed=1):
        base = self.P.GridTransform.cube(res, (-1.0, -1.0, -1.0), 2.0)
        return [(t.resolution, t.world_min, t.voxel_size, b)
                for t, b in self.P.build_dense_cascade(kind, base, levels, seed=seed)]

    def camera_rays(self, pos, w, h, first, count):
        return self.P.Camera(pos, (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, w, h).rays(first, count)

    def probe_rays(self, level, n, seed):
        return self.P.make_probe_rays(self.P.GridTransform(*level[:3]), n, seed)


class RefGen:
    """Input generation through the UNMODIFIED reference generators (oracle/_ref/libsogref.so:
    scene_gen.hpp, camera.hpp, bench.hpp make_probe_rays) -- the reference arm, which must not
    load the product library."""

    def __init__(self):
        from oracle_bindings import RefLib

        self.R = RefLib()

    def scene(self, kind, res, seed=1, count=12, fraction=0.05):
        g = self.R.scene(kind, res, seed=seed, fraction=fraction, count=count)
        return [(g.res, g.wmin, g.voxel, g.bits)], float(np.unpackbits(g.bits).sum()) / float(res ** 3)

    def cascade(self, kind, res, levels, seed=1):
        return [(g.res, g.wmin, g.voxel, g.bits) for g in self.R.cascade(kind, levels, res, seed=seed)]

    def camera_rays(self, pos, w, h, first, count):
        return self.R.camera_rays(pos, (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, w, h)[first:first + count]

    def probe_rays(self, level, n, seed):
        from oracle_bindings import Grid

        return self.R.probe_rays(Grid(level[0], level[1], level[2], level[3]), n, seed)


class Workload:
    """Grids (per object, as (resolution, world_min, voxel, bits) levels), the schedule, and
    the rays of every (step, object, rank) -- the same inputs in both arms."""

    def __init__(self, name: str, gen):
        self.name, self.gen = name, gen
        self.ray_order = 0
        self.cascade = False
        vox128 = 2.0 / 128
        self.schedule = (0, 0.5 * vox128, 0.0)  # (kind, dt0, growth)
        self.width = self.height = 800
        self.n_probe = 0
        if name == "cfg2":
            self.objects = []
            for kind, kw in CFG2_OBJECTS:
                lv, occ = gen.scene(kind, 128, **kw)
                self.objects.append(dict(label=f"{kind}:{kw}", levels=lv, occupancy=occ,
                                         scene=(kind, kw.get("seed", 1), kw.get("count", 12))))
        elif name == "cfg1":
            lv, occ = gen.scene("shell", 128, seed=1)
            self.objects = [dict(label="shell s1", levels=lv, occupancy=occ, scene=("shell", 1, 12))]
        elif name == "cfg3":
            lv = gen.cascade("blobs", 128, 4, seed=1)
            self.objects = [dict(label="blobs s1 x4 cascade", levels=lv, occupancy=None, scene=("blobs", 1, 12))]
            self.cascade = True
            self.width, self.height = 1297, 840
            self.schedule = (1, 0.5 * vox128, 1.0 / 256.0)
        elif name == "cfg4":
            lv, occ = gen.scene("blobs", 512, seed=1)
            self.objects = [dict(label="blobs s1 512^3", levels=lv, occupancy=occ, scene=None)]
            self.schedule = (0, 0.5 * 2.0 / 512, 0.0)
            self.n_probe = 1 << 24
            self.ray_order = 1  # incoherent probe rays: pass 1 bins them (sogk_sampler_set_ray_order)
        else:
            raise SystemExit(f"unknown config {name}")
        self.desc = DESC[name]
        self._probe_cache = {}

    def frame_rays(self) -> int:
        """Rays of one object per step before sharding."""
        return self.n_probe if self.name == "cfg4" else self.width * self.height

    def shard(self, step: int, obj: int, rank: int, world: int) -> dict:
        """The rays of (global step, object) for this rank: cfg2 -> one whole orbit view per rank
        (weak scaling); cfg1/3/4 -> a contiguous ceil(N/G) range of the step's rays (SURVEY
        §8e), ray_indices global (first = the range start)."""
        if self.name == "cfg2":
            view = view_of(step, rank, world, N_VIEWS, obj * (N_VIEWS // len(self.objects)))
            return dict(kind="camera", pos=orbit_pos(view), first=0, count=self.width * self.height)
        a, b = shard_range(self.frame_rays(), world, rank)
        if self.name == "cfg4":
            return dict(kind="probe", seed=1000 + step, first=a, count=b - a)
        return dict(kind="camera", pos=orbit_pos(0), first=a, count=b - a)

    def rays_per_object(self, world: int = 1, rank: int = 0) -> int:
        return self.shard(0, 0, rank, world)["count"]

    def host_rays(self, spec: dict) -> np.ndarray:
        if spec["kind"] == "camera":
            return self.gen.camera_rays(spec["pos"], self.width, self.height, spec["first"], spec["count"])
        key = spec["seed"]
        if key not in self._probe_cache:
            if len(self._probe_cache) > 2:
                self._probe_cache.clear()
            self._probe_cache[key] = self.gen.probe_rays(self.objects[0]["levels"][-1], self.n_probe, key)
        return self._probe_cache[key][spec["first"]:spec["first"] + spec["count"]]

    def fill_rays(self, P, out, spec: dict):
        """GPU arm: the rays of `spec` into the CUDA tensor `out` (camera rays by the raygen
        kernel, bit-identical to the host generator)."""
        if spec["kind"] == "camera":
            cam = P.Camera(spec["pos"], (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, self.width, self.height)
            cam.rays_device(spec["first"], spec["count"], out=out)
        else:
            import torch

            out.copy_(torch.from_numpy(np.ascontiguousarray(self.host_rays(spec))))

    # product-side helpers for the measurement tools (tools/prof_step.py, issue_probe.py)
    def dense_levels(self, P, obj: int):
        return [P.DenseGrid(P.GridTransform(r, w, v), b) for r, w, v, b in self.objects[obj]["levels"]]

    def step_schedule(self, P):
        return P.StepSchedule(*self.schedule)

    def device_rays(self, P, step: int, obj: int, rank: int = 0, world: int = 1):
        import torch

        spec = self.shard(step, obj, rank, world)
        out = torch.empty((spec["count"], 8), dtype=torch.float64, device="cuda")
        self.fill_rays(P, out, spec)
        return out

    def camera(self, P, spec: dict):
        return P.Camera(spec["pos"], (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, self.width, self.height)


def host_expand_link_bytes() -> int:
    """PCIe bytes per sample of the north-star outputs through sogk_sample_host: t_starts always;
    t_ends (8) and ray_indices (4) unless expanded on host threads (SOGK_HOST_EXPAND, sogk_api.cpp)."""
    e = os.environ.get("SOGK_HOST_EXPAND", "t")
    mode = 0 if e.startswith("0") else 1 if e.startswith("r") else 2 if e.startswith("t") else 3
    return 8 + (0 if mode & 2 else 8) + (0 if mode & 1 else 4)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
VARIANT_NAMES = {"hdda_skip": "sparse+hdda+skip", "dda_branch": "dense+dda+branch",
                 "dda_skip": "dense+dda+skip", "cd_skip": "dense+cd+skip"}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2404_10272_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one GPU per rank; ranks beyond the visible devices share them (tests: 2 ranks on 1 GPU)
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.backend)

    wl = Workload(args.config, ProductGen(P))
    sched = P.StepSchedule(*wl.schedule)
    n_obj = len(wl.objects)
    # --- grids: rank 0's payloads broadcast once over NVLink (NCCL), VDB built per rank (K1)
    grids = []
    build_ms = []
    dist_ms = []
    dist_grids = []
    for o in wl.objects:
        dense_lv, vdb_lv, cd_lv = [], [], []
        for res, wmin, voxel, bits in o["levels"]:
            t = P.GridTransform(res, wmin, voxel)
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
    dense_bytes = [sum(int(b.size) for *_, b in o["levels"]) for o in wl.objects]

    variants = {
        "hdda_skip": (P.Analyzer.hdda, P.KernelKind.skip),
        "dda_branch": (P.Analyzer.dda, P.KernelKind.branch),
        "dda_skip": (P.Analyzer.dda, P.KernelKind.skip),
        "cd_skip": (P.Analyzer.cd, P.KernelKind.skip),
    }
    if args.variants:
        variants = {k: v for k, v in variants.items() if k in args.variants.split(",")}
    def make_sampler(vname, i):
        an, kk = variants[vname]
        return P.Sampler(grids[i][1] if an == P.Analyzer.hdda else dist_grids[i] if an == P.Analyzer.cd
                         else grids[i][0], an, kk, sched, cascade=wl.cascade, ray_order=wl.ray_order)

    samplers = {vname: [make_sampler(vname, i) for i in range(n_obj)] for vname in variants}

    steps_total = args.warmup + args.steps
    specs = [[wl.shard(s, o, rank, world) for o in range(n_obj)] for s in range(steps_total)]
    nr = specs[0][0]["count"]  # this rank's rays per object per step
    # --- rays for every (step, object) in HBM before timing
    rays = [[torch.empty((nr, 8), dtype=torch.float64, device=dev) for _ in range(n_obj)]
            for _ in range(steps_total)]
    for s in range(steps_total):
        for o in range(n_obj):
            wl.fill_rays(P, rays[s][o], specs[s][o])
    torch.cuda.synchronize()
    base0 = specs[0][0]["first"]  # global index of this rank's first ray (same every step)

    # parts: the units one count/write pair processes -- one per object, or, for single-object
    # configs on several streams, one contiguous ray range per stream (each its own packed batch)
    # (--chunk-rays caps a part's rays: its pass-1 run slabs then stay L2-resident until pass 2
    # reads them, and the next chunk's pass 1 rewrites the same workspace lines in L2)
    k_obj = args.streams if (n_obj == 1 and args.streams > 1) else 1
    if args.chunk_rays > 0:
        k_obj = max(k_obj, -(-nr // args.chunk_rays))
    cut = [nr * i // k_obj for i in range(k_obj + 1)]
    parts = [(o, cut[i], cut[i + 1]) for o in range(n_obj) for i in range(k_obj)]
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

    stream = torch.cuda.current_stream()
    results = {}
    launches_per_step = {}
    for vname, smp in samplers.items():
        def one_step(s, ev=None):
            for pi, (o, a, b) in enumerate(parts):
                if ev is not None:
                    ev[pi][0].record(stream)
                smp[o].count(prays(s, pi), packed_info=packed[pi], stats=stats[pi])
                if ev is not None:
                    ev[pi][1].record(stream)
                smp[o].write(prays(s, pi), packed[pi], totals[(vname, s, pi)], ray_index_base=base0 + a,
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

            # parts -> streams: longest-processing-time first over the one-stream leg's per-part
            # times, so the streams' loads are even (objects differ ~4x in cost)
            part_ms = [sum(evs[k][pi][0].elapsed_time(evs[k][pi][2]) for k in range(args.steps))
                       for pi in range(n_parts)]
            load = [0.0] * args.streams
            assign = [0] * n_parts
            for pi in sorted(range(n_parts), key=lambda i: -part_ms[i]):
                j = min(range(args.streams), key=lambda x: load[x])
                assign[pi] = j
                load[j] += part_ms[pi]
            if not args.balance:
                assign = [pi % args.streams for pi in range(n_parts)]

            def step_overlapped(s):
                for pi, (o, a, b) in enumerate(parts):
                    st = side[assign[pi]]
                    smp[o].count(prays(s, pi), packed_info=packed[pi], stats=stats[pi], stream=st)
                    smp[o].write(prays(s, pi), packed[pi], totals[(vname, s, pi)], ray_index_base=base0 + a,
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
        results[vname] = dict(ms=ms, ms_serial=ms_serial, count_ms=count_ms, write_ms=write_ms, samples=samples,
                              clocks=clk.summary())
        # our kernels per count/write pair: count + scan (+ bin_count, scan, bin_scatter when the
        # rays are binned) and gather + tail
        launches_per_step[vname] = n_parts * (4 + (3 if wl.ray_order else 0))

    # --- parity of what was timed: the first timed step of every variant, re-run untimed
    # (same inputs, same kernels) and kept for the reference check in the cpu_baseline leg
    keep = {}
    if world == 1 and not args.no_cpu_baseline:
        s_chk = args.warmup
        for vname, smp in samplers.items():
            per_obj = []
            for o in range(n_obj):
                d = rays[s_chk][o]
                out = smp[o].sample(d, ray_index_base=base0, with_counters=False)
                stride = args.parity_stride
                idx = torch.arange(0, nr, stride, device=dev)
                pk = out.packed_info[idx]
                cnt = pk[:, 1]
                if int(cnt.sum().item()) > 0:
                    rep = torch.repeat_interleave(pk[:, 0], cnt)
                    off = torch.repeat_interleave(torch.cumsum(cnt, 0) - cnt, cnt)
                    g = rep + (torch.arange(int(cnt.sum().item()), device=dev) - off)
                else:
                    g = torch.zeros(0, dtype=torch.int64, device=dev)
                per_obj.append(dict(
                    counts=cnt.cpu().numpy(), status=out.status[idx].cpu().numpy(),
                    t_starts=out.t_starts[g].cpu().numpy(), t_ends=out.t_ends[g].cpu().numpy(),
                    ray_indices=out.ray_indices[g].cpu().numpy(),
                    cells=out.cells[g].cpu().numpy().view(np.uint32)))
                del out
            keep[vname] = per_obj
        torch.cuda.synchronize()

    if args.dump:  # every rank's outputs of the first timed step (tests: rank-count invariance)
        os.makedirs(args.dump, exist_ok=True)
        smp = samplers[next(iter(samplers))]
        for o in range(n_obj):
            out = smp[o].sample(rays[args.warmup][o], ray_index_base=base0)
            np.savez(os.path.join(args.dump, f"rank{rank}_obj{o}.npz"), first=base0,
                     packed_info=out.packed_info.cpu().numpy(), t_starts=out.t_starts.cpu().numpy(),
                     t_ends=out.t_ends.cpu().numpy(), ray_indices=out.ray_indices.cpu().numpy(),
                     cells=out.cells.cpu().numpy(), status=out.status.cpu().numpy())
        torch.cuda.synchronize()

    P.release_workspaces()
    # --- render leg: render_frame (pass 1 + pass 2 on the camera rays, shading + compositing),
    # the paper's rendered-frames metric; one frame = one object's view (this rank's pixels)
    render = None
    if not args.no_render and wl.name != "cfg4":
        scenes = [P.analytic_scene(o["scene"][0], P.GridTransform(*o["levels"][0][:3]), seed=o["scene"][1],
                                   count=o["scene"][2]) for o in wl.objects]
        r_res = torch.empty((nr, 5), dtype=torch.float64, device=dev)
        r_rgb = torch.empty((nr, 3), dtype=torch.uint8, device=dev)
        r_st = torch.zeros(8, dtype=torch.int64, device=dev)
        render = {}
        for vname, smp in samplers.items():
            def rstep(s_):
                for o in range(n_obj):
                    sp = specs[s_][o]
                    cam = wl.camera(P, sp)._c()
                    P._check(P.lib.sogk_render_camera(smp[o]._h, scenes[o].handle, P.C.byref(cam), sp["first"],
                                                      sp["count"], r_res.data_ptr(), r_rgb.data_ptr(),
                                                      r_st.data_ptr(), stream.cuda_stream or None), "render")
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
                             "mpix_per_sec": frames * nr / (rms / 1e3) / 1e6}

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
        # units of host work: one object each (worker w takes objects w, w + W, ...), or, for a
        # single-object config, one contiguous ray range per worker with its own sampler (a sampler
        # serialises its host calls); capacities from an untimed count of every step
        if n_obj == 1 and args.e2e_workers > 1:
            W = min(args.e2e_workers, 2)  # measured: 2 ranges beat 4 (cfg1 44.6 vs 40.1, cfg4 143 vs 112 Mrays/s)
            cut = [nr * i // W for i in range(W + 1)]
            caps = [0] * W
            pk = torch.empty((nr, 2), dtype=torch.int64, device=dev)
            st_ = torch.zeros(8, dtype=torch.int64, device=dev)
            for s_ in range(steps_total):  # per-range sample totals (untimed sizing)
                smp[0].count(rays[s_][0], packed_info=pk, stats=st_)
                cs = torch.cumsum(pk[:, 1], 0).cpu().numpy()
                for i in range(W):
                    tot_i = int(cs[cut[i + 1] - 1] - (cs[cut[i] - 1] if cut[i] > 0 else 0)) if cut[i + 1] > cut[i] else 0
                    caps[i] = max(caps[i], tot_i)
            units = [(make_sampler(vname0, 0) if i else smp[0], 0, cut[i], cut[i + 1], caps[i]) for i in range(W)]
            n_workers = W
        else:
            units = [(smp[o], o, 0, nr, max(obj_cap)) for o in range(n_obj)]
            n_workers = max(1, min(args.e2e_workers, n_obj))
        P.release_workspaces()
        hcap = max(1, max(u[4] for u in units))
        urays = max(u[3] - u[2] for u in units)

        def host_outputs():  # pinned output buffers, one set per worker thread
            o = dict(packed_info=torch.empty((urays, 2), dtype=torch.int64, pin_memory=True).numpy(),
                     t_starts=torch.empty(hcap, dtype=torch.float64, pin_memory=True).numpy(),
                     t_ends=torch.empty(hcap, dtype=torch.float64, pin_memory=True).numpy(),
                     ray_indices=torch.empty(hcap, dtype=torch.int32, pin_memory=True).numpy(),
                     stats=np.zeros(8, np.int64))
            o["counters"] = torch.empty((urays, 3), dtype=torch.int32, pin_memory=True).numpy()
            return o

        h_outs = [host_outputs() for _ in range(n_workers)]
        lib = P.lib
        pool = ThreadPoolExecutor(n_workers) if n_workers > 1 else None

        def e2e_objects(s, full, w):
            # full: the north-star packed intervals (packed_info, t_starts, t_ends, ray_indices);
            # lean: what the reference's run_sampler returns per ray (sampling.hpp:157-164), its
            # sample buffer (packed t_starts + packed_info) and its three counters.  Worker w
            # takes units w, w + W, ... (independent samplers: each call is synchronous and
            # pipelines its own chunks; ctypes drops the GIL, so calls overlap)
            h_out = h_outs[w]
            for u in range(w, len(units), n_workers):
                sm, o, a, b, cap_u = units[u]
                rc = lib.sogk_sample_host(sm._h, h_rays[s][o].data_ptr() + a * 64, b - a, base0 + a, hcap,
                                          h_out["packed_info"].ctypes.data, h_out["t_starts"].ctypes.data,
                                          h_out["t_ends"].ctypes.data if full else None,
                                          h_out["ray_indices"].ctypes.data if full else None,
                                          None, None, None,
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

        e2e_full_s = timed(True)
        e2e_lean_s = timed(False)
        samples0 = sum(totals[(vname0, args.warmup + k, pi)] for k in range(args.steps) for pi in range(n_parts))
        if pool is not None:
            pool.shutdown()
        e2e = dict(full_seconds=e2e_full_s, lean_seconds=e2e_lean_s, h2d=nr * 64 * n_obj, workers=n_workers,
                   # t_ends / ray_indices are expanded on host threads from the downloaded
                   # t_starts + packed_info (sogk_sample_host, SOGK_HOST_EXPAND): not on the link
                   full_d2h=samples0 * host_expand_link_bytes() / args.steps + nr * 16 * n_obj,
                   lean_d2h=samples0 * 8 / args.steps + nr * (16 + 12) * n_obj)

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
                          rays=rsum(nr * n_obj * args.steps), count_ms=r["count_ms"], write_ms=r["write_ms"],
                          local_samples=r["samples"], clocks=r["clocks"])
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    head = "hdda_skip" if "hdda_skip" in agg else next(iter(agg))
    h = agg[head]
    total_rays = h["rays"]  # every rank's rays of the timed steps
    sec = h["ms"] / 1e3
    rays_s = total_rays / sec
    samples_s = h["samples"] / sec
    peak, peak_src = load_peaks()
    # roofline: dominant kernel (larger share of the step) with its algorithmic bytes
    # (SURVEY §8(d)): pass 1 reads the rays (64 B) and writes packed_info (16 B) per ray;
    # pass 2 reads packed_info (16 B/ray) and writes the samples (24 B each).  The slabs
    # pass 1 hands to pass 2 are not algorithmic; ncu's DRAM bytes (`traffic`,
    # profiles/traffic_<cfg>.json) show them.
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
        "metric": METRIC,
        "value": rays_s,
        "unit": "rays/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": h["ms"] / args.steps,
        "higher_is_better": True,
        "scaling": scaling_of(args.config),
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (procedural occupancy grids from the reference generators, camera/probe rays)",
        "config": workload_config(args.config, world, args.streams),
        "samples_per_sec": samples_s,
        "samples_per_step": h["samples"] / args.steps,
        "gpu_launches": launches_per_step[head] * args.steps,
        "clocks": h["clocks"],
    }
    if e2e:
        line["e2e"] = {"value": total_rays / e2e["full_seconds"], "unit": "rays/s",
                       "h2d_bytes_per_step": int(e2e["h2d"]), "d2h_bytes_per_step": int(e2e["full_d2h"]),
                       "api": "sogk_sample_host: pinned host rays in; out the north-star packed intervals "
                              "(packed_info, t_starts, t_ends, ray_indices) in host memory; "
                              f"{host_expand_link_bytes()} PCIe bytes per sample (SOGK_HOST_EXPAND: t_ends = "
                              "t + step(t) and/or ray_indices expanded on host threads from the downloaded "
                              "t_starts / packed_info while later chunks are in flight)",
                       "host_threads": e2e["workers"],
                       "lean": {"value": total_rays / e2e["lean_seconds"], "unit": "rays/s",
                                "d2h_bytes_per_step": int(e2e["lean_d2h"]),
                                "outputs": "what run_sampler returns per ray (sampling.hpp:157-164): "
                                           "packed t_starts + packed_info + the three counters"}}
    line["roofline"] = {
        "bound": "hbm", "kernel": dom["kernel"], "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "traffic": traffic.get(dom_key, {}).get("dram_bytes_per_launch"),
        "peak_source": peak_src, "algorithmic_bytes_per_launch": dom["bytes"] / launches,
        "note": "pass 1 is bound by traversal issue/latency, not HBM (DESIGN.md §4); traffic = ncu "
                "dram read+write of one launch (object 0), " + traffic.get("source", "no capture committed"),
        "other_pass": {"kernel": other["kernel"], "achieved": gbs(other), "frac": gbs(other) / peak,
                       "algorithmic_bytes_per_launch": other["bytes"] / launches,
                       "traffic": traffic.get(other_key, {}).get("dram_bytes_per_launch")},
        "issue_ceiling": issue}
    if world == 1 and not args.no_cpu_baseline:
        cb, parity = cpu_baseline_and_parity(wl, args, keep, base0)
        line["cpu_baseline"] = cb
        line["parity"] = parity
    line.update({
        "variants": {k: {"rays_per_sec": v["rays"] / (v["ms"] / 1e3),
                         "samples_per_sec": v["samples"] / (v["ms"] / 1e3),
                         "ms_per_step": v["ms"] / args.steps,
                         "ms_per_step_one_stream": v["ms_serial"] / args.steps,
                         "count_ms_per_step": v["count_ms"] / args.steps,
                         "write_ms_per_step": v["write_ms"] / args.steps} for k, v in agg.items()},
        "hdda_vs_dda_branch": (agg["dda_branch"]["ms"] / agg["hdda_skip"]["ms"]) if {"dda_branch", "hdda_skip"} <= agg.keys() else None,
        "step_roofline": {"bytes_per_step": step_bytes / args.steps, "achieved_gbs": step_gbs,
                          "frac": step_gbs / peak,
                          "basis": "N_rays*(64+16) + N_samples*24 + VDB bytes (SURVEY §8d)"},
        "vdb_build_ms": build_ms,
        "distance_build_ms": dist_ms,
        "grid_bytes": {"dense": dense_bytes, "vdb_sog1": vdb_bytes},
        "render": ({"what": "render_frame on the GPU (pass 1 + pass 2 on the camera rays, per-sample "
                            "shading, per-ray composite_detailed + Image::set_pixel), "
                            f"{wl.width}x{wl.height} frames ({nr} pixels per rank), rank 0",
                    "variants": render} if render else None),
    })
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref: the unmodified reference headers) -- the cpu_baseline leg and the
# reference arm; the only places bench.py loads anything under oracle/
# ---------------------------------------------------------------------------
def _ref_levels(o):
    from oracle_bindings import Grid

    return [Grid(tuple(r), tuple(w), v, b) for r, w, v, b in o["levels"]]


def _ref_samplers(wl, analyzer, kernel):
    from oracle_bindings import RefLib

    R = RefLib()
    k, dt0, gr = wl.schedule
    return R, [R.sampler(_ref_levels(o), analyzer, kernel, k, dt0, gr, cascade=wl.cascade) for o in wl.objects]


def _spin_masks(wl, rays_per_obj):
    """Rays on which the reference HDDA never returns are screened out with the
    capped oracle detector; they are excluded from the CPU timing and counted."""
    from oracle_bindings import HDDA, SKIP, Oracle

    O = Oracle()
    k, dt0, gr = wl.schedule
    masks = []
    for o, r in zip(wl.objects, rays_per_obj):
        s = O.sampler(_ref_levels(o), HDDA, SKIP, k, dt0, gr, cascade=wl.cascade)
        masks.append((O.sample(s, r).status == 2).astype(np.uint8))
    return masks


def _strided_rays(wl, stride, step, rank=0, world=1):
    return [np.ascontiguousarray(wl.host_rays(wl.shard(step, o, rank, world))[::stride])
            for o in range(len(wl.objects))]


def cpu_baseline_and_parity(wl, args, keep, base0):
    """cpu_baseline: the unmodified reference sampler (oracle/_ref) timed on the host cores
    over a strided sample of step 0's rays.  parity: the GPU outputs of the first timed step
    (every variant bench timed) on a strided subset of its rays against the reference's
    run_sampler on the same rays -- counts, t_starts, t_ends, ray_indices and cells bit for bit."""
    from oracle_bindings import BRANCH, CD, DDA, HDDA, SKIP

    try:
        R, smp = _ref_samplers(wl, HDDA, SKIP)
    except FileNotFoundError:
        return ({"value": None, "unit": "rays/s", "kind": "reference", "cores": 0,
                 "sample": "oracle/_ref missing"}, {"status": "unchecked (oracle/_ref missing)"})
    cores = os.cpu_count() or 1
    stride = args.cpu_stride
    rays = _strided_rays(wl, stride, 0)
    masks = _spin_masks(wl, rays)
    sec, n = 0.0, 0
    for s, r, m in zip(smp, rays, masks):
        dt, _ = s.time(r, skip=m, threads=cores, reps=1)
        sec += dt
        n += int(r.shape[0] - m.sum())
    cb = {"value": n / sec, "unit": "rays/s", "cores": cores, "kind": "reference",
          "sample": f"sparse+hdda+skip via sog::run_sampler, every {stride}th ray of step 0 "
                    f"({n} rays over {len(rays)} object(s)), {cores} threads, spin-screened "
                    f"{int(sum(m.sum() for m in masks))} rays"}
    # parity on the first timed step
    an_k = {"hdda_skip": (HDDA, SKIP), "dda_branch": (DDA, BRANCH), "dda_skip": (DDA, SKIP), "cd_skip": (CD, SKIP)}
    ps = args.parity_stride
    prays = _strided_rays(wl, ps, args.warmup)
    pmasks = _spin_masks(wl, prays)
    checked, bad, rays_checked, samples_checked, screened = [], [], 0, 0, 0
    for vname, per_obj in keep.items():
        an, k = an_k[vname]
        _, rs = _ref_samplers(wl, an, k)
        for o, (s, r, m, got) in enumerate(zip(rs, prays, pmasks, per_obj)):
            und = (got["status"] == 2).astype(np.uint8)
            skip = np.maximum(m, und)
            want = s.sample(r, skip=skip, threads=cores)
            ok_rays = skip == 0
            gc = np.where(ok_rays, got["counts"], 0)
            wc = want.packed_info[:, 1]
            sel = np.repeat(ok_rays, got["counts"])
            ri_want = np.repeat(np.arange(r.shape[0], dtype=np.int64) * ps + base0, wc).astype(np.int32)
            same = (np.array_equal(gc, wc)
                    and np.array_equal(got["t_starts"][sel].view(np.uint64), want.t_starts.view(np.uint64))
                    and np.array_equal(got["t_ends"][sel].view(np.uint64), want.t_ends.view(np.uint64))
                    and np.array_equal(got["ray_indices"][sel], ri_want)
                    and np.array_equal(got["cells"][sel], want.cells))
            rays_checked += int(ok_rays.sum())
            samples_checked += int(wc.sum())
            screened += int(skip.sum())
            (checked if same else bad).append(f"{VARIANT_NAMES[vname]}:{wl.objects[o]['label']}")
    parity = {"status": "bit-exact" if not bad and checked else ("MISMATCH" if bad else "unchecked"),
              "against": "oracle/_ref (the unmodified reference run_sampler / run_cascade_sampler)",
              "step": args.warmup, "ray_stride": ps, "rays_checked": rays_checked,
              "samples_checked": samples_checked, "spin_screened_rays": screened,
              "outputs": "per-ray counts, t_starts, t_ends, ray_indices, cells (bit-exact)",
              "cases_ok": len(checked), "cases_bad": bad}
    return cb, parity


def run_reference(args):
    """--impl reference: the reference CPU sampler (oracle/_ref, the unmodified headers) on the
    host cores, inputs generated by the reference's own generators; the product library is
    never loaded in this process."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle_bindings import HDDA, SKIP

    try:
        wl = Workload(args.config, RefGen())
        R, smp = _ref_samplers(wl, HDDA, SKIP)
    except FileNotFoundError as e:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not built: {e}"}))
        return
    cores = os.cpu_count() or 1
    stride = args.cpu_stride
    step_rays, step_masks = [], []
    for s in range(args.warmup + args.steps):
        r, m = [], []
        for rk in range(world):  # the whole job's rays of this step (every rank's share)
            rr = _strided_rays(wl, stride, s, rk, world)
            r += rr
            m += _spin_masks(wl, rr)
        step_rays.append(r)
        step_masks.append(m)
    per_step_rays = [sum(int(x.shape[0] - m.sum()) for x, m in zip(r, mm)) for r, mm in zip(step_rays, step_masks)]
    n_obj = len(wl.objects)

    def step(s):
        t = 0.0
        for i, (r, m) in enumerate(zip(step_rays[s], step_masks[s])):
            dt, _ = smp[i % n_obj].time(r, skip=m, threads=cores, reps=1)
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
    sample = (f"every {stride}th ray of each step's rays (all ranks' shares), sog::run_sampler "
              f"(sparse+hdda+skip) on {cores} threads, inputs from the reference generators, "
              f"spin-screened {sum(int(m.sum()) for mm in step_masks for m in mm)} rays")
    line = {
        "impl": "reference", "metric": METRIC,
        "value": v, "unit": "rays/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_s / args.steps * 1e3, "higher_is_better": True,
        "scaling": scaling_of(args.config), "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (procedural occupancy grids from the reference generators, camera/probe rays)",
        "config": workload_config(args.config, world, args.streams),
        "cpu_baseline": {"value": v, "unit": "rays/s", "cores": cores, "kind": "reference", "sample": sample},
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
    ap.add_argument("--parity-stride", type=int, default=64,
                    help="every k-th ray of the first timed step is checked against the reference")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-workers", type=int, default=4,
                    help="host threads issuing sogk_sample_host calls concurrently (objects, or ray ranges of one object)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    ap.add_argument("--streams", type=int, default=2,
                    help="CUDA streams the step's objects are spread over (1: one stream)")
    ap.add_argument("--balance", type=int, default=0,
                    help="1: assign parts to streams by measured cost (LPT); 0: round robin")
    ap.add_argument("--chunk-rays", type=int, default=0,
                    help="at most this many rays per count/write pair (0: one pair per object or stream part)")
    ap.add_argument("--backend", default="nccl", help="torch.distributed backend under torchrun (tests: gloo)")
    ap.add_argument("--dump", default="", help="directory: every rank saves its outputs of the first timed step")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = {"cfg1": 200, "cfg2": 50, "cfg3": 200, "cfg4": 10}[args.config]
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
