"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  -> oracle/_build/libsog_oracle.so, the plain-C restatement of the
  reference path (oracle/sog_oracle.c).
* ``RefLib``  -> oracle/_ref/libsogref.so, the unmodified reference headers behind
  a C shim (oracle/ref_shim.cpp).  Built only where /root/reference exists; the
  prebuilt .so travels to the GPU box with the repo snapshot.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libsog_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libsogref.so")

DDA, HDDA, CD = 0, 1, 2
BRANCH, SKIP = 0, 1
CONSTANT, LINEAR = 0, 1
SCENE_KINDS = {"blobs": 0, "shell": 1, "sponge": 2, "random": 3}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build_checkers() -> None:
    """Compile oracle/ (and oracle/_ref when /root/reference is present)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


@dataclass
class Grid:
    """Host description of one dense grid level (transform + bit payload)."""

    res: tuple
    wmin: tuple
    voxel: float
    bits: np.ndarray  # uint8, ceil(N/8), x-fastest LSB-first (grid.hpp:117-124)

    @property
    def nbytes(self) -> int:
        return int(self.bits.size)


class _OgEvent(C.Structure):
    _fields_ = [("ijk", C.c_int32 * 3), ("level", C.c_int32), ("t0", C.c_double),
                ("t1", C.c_double), ("occupied", C.c_int32), ("grid_level", C.c_int32)]


class _OgSampler(C.Structure):
    _fields_ = [("levels", C.c_void_p * 8), ("n_levels", C.c_int32), ("cascade", C.c_int32),
                ("analyzer", C.c_int32), ("kernel", C.c_int32), ("sched_kind", C.c_int32),
                ("dt0", C.c_double), ("growth", C.c_double), ("spin_cap", C.c_int32)]


@dataclass
class Packed:
    packed_info: np.ndarray
    t_starts: np.ndarray
    t_ends: np.ndarray
    ray_indices: np.ndarray
    cells: np.ndarray
    levels: np.ndarray
    counters: np.ndarray
    status: np.ndarray

    @property
    def total(self) -> int:
        return int(self.t_starts.size)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_checkers()
        L = C.CDLL(path)
        self.L = L
        L.og_dense_create.restype = C.c_void_p
        L.og_dense_create.argtypes = [_i32p, _dp, C.c_double, _u8p]
        L.og_sparse_build.restype = C.c_void_p
        L.og_sparse_build.argtypes = [C.c_void_p]
        L.og_distance_build.restype = C.c_void_p
        L.og_distance_build.argtypes = [C.c_void_p]
        L.og_distance_data.restype = C.c_void_p
        L.og_distance_data.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        L.og_grid_free.argtypes = [C.c_void_p]
        L.og_sparse_serialize.restype = C.c_int64
        L.og_sparse_serialize.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.og_sparse_leaf_count.restype = C.c_int64
        L.og_sparse_leaf_count.argtypes = [C.c_void_p]
        L.og_dense_voxel_at.restype = C.c_int32
        L.og_dense_voxel_at.argtypes = [C.c_void_p, _i32p]
        L.og_sparse_query.restype = C.c_int32
        L.og_sparse_query.argtypes = [C.c_void_p, _i32p, C.POINTER(C.c_int32), _i32p,
                                      C.POINTER(C.c_int32)]
        L.og_collect_events.restype = C.c_int64
        L.og_collect_events.argtypes = [C.POINTER(_OgSampler), _dp, C.c_int64,
                                        C.POINTER(_OgEvent), _i64p]
        L.og_sample_ray.restype = C.c_int64
        L.og_sample_batch.restype = C.c_int64
        L.og_sample_batch.argtypes = [C.POINTER(_OgSampler), _dp, C.c_int64, C.c_int64,
                                      C.c_int64, _i64p, _dp, _dp, _i32p, _u32p, _u8p, _i32p, _u8p]
        L.og_composite.argtypes = [_dp, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, _dp,
                                   C.c_int32, C.c_double, C.c_double, _dp]
        L.og_set_pixel.argtypes = [_dp, _u8p]
        L.og_psnr.restype = C.c_double
        L.og_psnr.argtypes = [_u8p, _u8p, C.c_int64]
        self._owned = []

    # compositing (render.hpp) --------------------------------------------------
    @staticmethod
    def _prims(prims) -> np.ndarray:
        """Primitives as the og_primitive layout (int32 shape + pad, then 14 doubles)."""
        dt = np.dtype([("shape", np.int32), ("pad", np.int32), ("center", np.float64, 3),
                       ("radius", np.float64), ("lo", np.float64, 3), ("hi", np.float64, 3),
                       ("density", np.float64), ("color", np.float64, 3)])
        a = np.zeros(max(1, len(prims)), dt)
        for i, p in enumerate(prims):
            a[i] = (p.shape, 0, p.center, p.radius, p.lo, p.hi, p.density, p.color)
        return a

    def composite(self, ray, samples, prims, background, sched_kind, dt0, growth=0.0) -> np.ndarray:
        """composite_detailed (render.hpp:97-118) -> [r, g, b, weight_sum, transmittance]."""
        out = np.zeros(5, np.float64)
        smp = np.ascontiguousarray(samples, np.float64)
        pa = self._prims(prims)
        self.L.og_composite(np.ascontiguousarray(ray, np.float64), smp.ctypes.data if smp.size else None,
                            smp.size, pa.ctypes.data, len(prims), np.asarray(background, np.float64),
                            sched_kind, dt0, growth, out)
        return out

    def set_pixel(self, rgb) -> np.ndarray:
        out = np.zeros(3, np.uint8)
        self.L.og_set_pixel(np.asarray(rgb, np.float64), out)
        return out

    # grids ----------------------------------------------------------------
    def dense(self, g: Grid) -> int:
        h = self.L.og_dense_create(np.asarray(g.res, np.int32), np.asarray(g.wmin, np.float64),
                                   float(g.voxel), np.ascontiguousarray(g.bits, np.uint8))
        self._owned.append(h)
        return h

    def sparse(self, g: Grid) -> int:
        d = self.dense(g)
        h = self.L.og_sparse_build(d)
        self._owned.append(h)
        return h

    def distance(self, g: Grid) -> int:
        d = self.dense(g)
        h = self.L.og_distance_build(d)
        self._owned.append(h)
        return h

    def distance_field(self, g: Grid):
        """build_distance (distance.hpp:45-103) -> (int32 [z][y][x], all_empty)."""
        h = self.distance(g)
        ae = C.c_int32(0)
        p = self.L.og_distance_data(h, C.byref(ae))
        n = int(g.res[0]) * int(g.res[1]) * int(g.res[2])
        a = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_int32)), shape=(n,)).copy()
        return a.reshape(g.res[2], g.res[1], g.res[0]), bool(ae.value)

    def sog1(self, g: Grid) -> bytes:
        s = self.sparse(g)
        n = self.L.og_sparse_serialize(s, None, 0)
        buf = (C.c_uint8 * n)()
        self.L.og_sparse_serialize(s, buf, n)
        return bytes(buf)

    def free(self):
        for h in reversed(self._owned):
            self.L.og_grid_free(h)
        self._owned.clear()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    # sampling -------------------------------------------------------------
    def sampler(self, levels, analyzer, kernel, sched_kind, dt0, growth=0.0, cascade=False,
                spin_cap=64) -> _OgSampler:
        s = _OgSampler()
        handles = [self.sparse(g) if analyzer == HDDA else self.distance(g) if analyzer == CD
                   else self.dense(g) for g in levels]
        for i, h in enumerate(handles):
            s.levels[i] = h
        s.n_levels = len(handles)
        s.cascade = 1 if cascade else 0
        s.analyzer, s.kernel, s.sched_kind = analyzer, kernel, sched_kind
        s.dt0, s.growth, s.spin_cap = float(dt0), float(growth), int(spin_cap)
        return s

    def sample(self, s: _OgSampler, rays: np.ndarray, ray_index_base: int = 0) -> Packed:
        rays = np.ascontiguousarray(rays, np.float64).reshape(-1, 8)
        n = rays.shape[0]
        cap = max(1024, 64 * n)
        while True:
            pi = np.zeros((n, 2), np.int64)
            ts = np.zeros(cap, np.float64)
            te = np.zeros(cap, np.float64)
            ri = np.zeros(cap, np.int32)
            ce = np.zeros(cap, np.uint32)
            lv = np.zeros(cap, np.uint8)
            ct = np.zeros((n, 3), np.int32)
            st = np.zeros(n, np.uint8)
            tot = self.L.og_sample_batch(C.byref(s), rays, n, ray_index_base, cap, pi, ts, te, ri,
                                         ce, lv, ct, st)
            if tot <= cap:
                return Packed(pi, ts[:tot], te[:tot], ri[:tot], ce[:tot], lv[:tot], ct, st)
            cap = int(tot)

    def events(self, s: _OgSampler, ray, cap: int = 1 << 16):
        evs = (_OgEvent * cap)()
        ctr = np.zeros(2, np.int64)
        n = self.L.og_collect_events(C.byref(s), np.ascontiguousarray(ray, np.float64), cap, evs,
                                     ctr)
        out = [(tuple(evs[i].ijk), evs[i].level, evs[i].t0, evs[i].t1, evs[i].occupied,
                evs[i].grid_level) for i in range(max(0, min(n, cap)))]
        return n, out, ctr


class RefLib:
    """The unmodified reference (oracle/_ref/libsogref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.ref_hardware_concurrency.restype = C.c_int
        L.ref_generate_scene.restype = C.c_double
        L.ref_generate_scene.argtypes = [C.c_int, _i32p, _dp, C.c_double, C.c_uint64, C.c_double,
                                         C.c_int, C.c_double, _u8p]
        L.ref_dense_cascade.argtypes = [C.c_int, _i32p, _dp, C.c_double, C.c_uint64, C.c_double,
                                        C.c_int, C.c_double, C.c_int, _u8p, _dp, _dp]
        L.ref_camera_rays.argtypes = [_dp, _dp, _dp, C.c_double, C.c_int, C.c_int, C.c_double, _dp]
        L.ref_probe_rays.argtypes = [_i32p, _dp, C.c_double, C.c_int, C.c_uint64, _dp]
        L.ref_random_rays.argtypes = [_i32p, _dp, C.c_double, C.c_int, C.c_uint64, _dp]
        L.ref_random_grid.argtypes = [_i32p, _dp, C.c_double, C.c_uint64, C.c_double, _u8p]
        L.ref_random_blocky_grid.argtypes = [_i32p, _dp, C.c_double, C.c_uint64, C.c_double,
                                             C.c_double, _u8p]
        L.ref_build_sog1.restype = C.c_int64
        L.ref_build_sog1.argtypes = [_i32p, _dp, C.c_double, _u8p, C.c_void_p, C.c_int64]
        L.ref_build_sparse_ms.restype = C.c_double
        L.ref_build_sparse_ms.argtypes = [_i32p, _dp, C.c_double, _u8p, C.c_int]
        L.ref_sampler_create.restype = C.c_void_p
        L.ref_sampler_create.argtypes = [C.c_int, C.c_int, _i32p, _dp, _dp, C.c_void_p, C.c_int,
                                         C.c_int, C.c_int, C.c_double, C.c_double]
        L.ref_sampler_free.argtypes = [C.c_void_p]
        L.ref_sample_batch.restype = C.c_int64
        L.ref_sample_batch.argtypes = [C.c_void_p, _dp, C.c_int64, C.c_void_p, C.c_int, C.c_int64,
                                       _i64p, _dp, _dp, _u32p, _u8p, _i32p]
        L.ref_collect_events.restype = C.c_int64
        L.ref_collect_events.argtypes = [C.c_void_p, _dp, C.c_int64, _i32p, _dp, _i64p]
        L.ref_build_distance.restype = C.c_int
        L.ref_build_distance.argtypes = [_i32p, _dp, C.c_double, _u8p, _i32p]
        L.ref_scene_primitives.restype = C.c_int
        L.ref_scene_primitives.argtypes = [C.c_int, _i32p, _dp, C.c_double, C.c_uint64, C.c_double,
                                           C.c_int, _dp, C.c_int, _dp]
        L.ref_render_frame.argtypes = [C.c_int, C.c_uint64, C.c_double, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _u8p,
                                       _i64p]
        L.ref_composite.argtypes = [_dp, C.c_void_p, C.c_int64, _dp, C.c_int, _dp, C.c_int,
                                    C.c_double, C.c_double, _dp]
        L.ref_run_matrix.restype = C.c_int64
        L.ref_run_matrix.argtypes = [C.c_int, C.c_uint64, C.c_double, C.c_int, C.c_int, C.c_int,
                                     C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int64]
        L.ref_time_sampler.restype = C.c_double
        L.ref_time_sampler.argtypes = [C.c_void_p, _dp, C.c_int64, C.c_void_p, C.c_int, C.c_int,
                                       C.POINTER(C.c_int64)]

    @staticmethod
    def _nbytes(res):
        return (int(res[0]) * int(res[1]) * int(res[2]) + 7) // 8

    def scene(self, kind, res=128, seed=1, fraction=0.05, count=12, threshold=0.01,
              wmin=(-1.0, -1.0, -1.0), extent=2.0) -> Grid:
        r = np.array([res] * 3 if np.isscalar(res) else res, np.int32)
        voxel = extent / float(r[0])
        bits = np.zeros(self._nbytes(r), np.uint8)
        self.L.ref_generate_scene(SCENE_KINDS[kind], r, np.asarray(wmin, np.float64), voxel, seed,
                                  fraction, count, threshold, bits)
        return Grid(tuple(int(x) for x in r), tuple(wmin), voxel, bits)

    def cascade(self, kind, levels=4, res=128, seed=1, fraction=0.05, count=12, threshold=0.01):
        r = np.array([res] * 3, np.int32)
        nb = self._nbytes(r)
        bits = np.zeros(nb * levels, np.uint8)
        wm = np.zeros(3 * levels, np.float64)
        vx = np.zeros(levels, np.float64)
        self.L.ref_dense_cascade(SCENE_KINDS[kind], r, np.array([-1.0] * 3), 2.0 / res, seed,
                                 fraction, count, threshold, levels, bits, wm, vx)
        return [Grid(tuple(int(x) for x in r), tuple(wm[3 * b:3 * b + 3]), float(vx[b]),
                     bits[b * nb:(b + 1) * nb].copy()) for b in range(levels)]

    def distance_field(self, g: Grid):
        """the reference build_distance -> (int32 [z][y][x], all_empty)."""
        out = np.zeros(int(g.res[0]) * int(g.res[1]) * int(g.res[2]), np.int32)
        ae = self.L.ref_build_distance(np.asarray(g.res, np.int32), np.asarray(g.wmin, np.float64),
                                       g.voxel, np.ascontiguousarray(g.bits, np.uint8), out)
        return out.reshape(g.res[2], g.res[1], g.res[0]), bool(ae)

    def scene_primitives(self, kind, res=128, seed=1, fraction=0.05, count=12,
                         wmin=(-1.0, -1.0, -1.0), extent=2.0):
        """generate_scene's AnalyticScene -> (array [n, 16], background[3])."""
        r = np.array([res] * 3, np.int32)
        out = np.zeros((512, 16), np.float64)
        bg = np.zeros(3, np.float64)
        n = self.L.ref_scene_primitives(SCENE_KINDS[kind], r, np.asarray(wmin, np.float64),
                                        extent / res, seed, fraction, count, out, 512, bg)
        return out[:n].copy(), bg

    def composite(self, ray, samples, prims16, background, sched_kind, dt0, growth=0.0):
        """the reference's composite_detailed; prims16 as returned by scene_primitives."""
        out = np.zeros(5, np.float64)
        smp = np.ascontiguousarray(samples, np.float64)
        pa = np.ascontiguousarray(prims16, np.float64).reshape(-1, 16)
        self.L.ref_composite(np.ascontiguousarray(ray, np.float64), smp.ctypes.data if smp.size else None,
                             smp.size, pa if pa.size else np.zeros(16), len(pa),
                             np.asarray(background, np.float64), sched_kind, dt0, growth, out)
        return out

    def render_frame(self, kind, seed=1, fraction=0.0, resolution=128, cascades=1, sched_kind=0,
                     width=160, height=120, grid=0, analyzer=0, kernel=0, threads=0):
        """render_frame (bench.hpp:424-461) of one variant on build_assets(cfg) ->
        (image HxWx3 uint8, lookups, steps, samples)."""
        rgb = np.zeros(width * height * 3, np.uint8)
        st = np.zeros(3, np.int64)
        nt = threads or max(1, self.L.ref_hardware_concurrency())
        self.L.ref_render_frame(SCENE_KINDS[kind], seed, fraction, resolution, cascades, sched_kind,
                                width, height, grid, analyzer, kernel, nt, rgb, st)
        return rgb.reshape(height, width, 3), int(st[0]), int(st[1]), int(st[2])

    def run_matrix(self, kind, seed=1, fraction=0.0, resolution=32, cascades=1, sched_kind=0,
                   width=32, height=24, repetitions=1):
        """the reference run_matrix (bench.hpp:514-553) -> (emit_json text, emit_csv text)."""
        cap = 1 << 16
        while True:
            buf = C.create_string_buffer(cap)
            n = self.L.ref_run_matrix(SCENE_KINDS[kind], seed, fraction, resolution, cascades,
                                      sched_kind, width, height, repetitions, buf, cap)
            if n > 0:
                j, c = buf.raw[:n - 1].split(b"\0", 1)
                return j.decode(), c.decode()
            cap = -n

    def camera_rays(self, pos=(1.9, 1.4, 2.3), target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0),
                    vfov=42.0, width=160, height=120, t_far=1e6) -> np.ndarray:
        out = np.zeros((width * height, 8), np.float64)
        self.L.ref_camera_rays(np.asarray(pos, np.float64), np.asarray(target, np.float64),
                               np.asarray(up, np.float64), vfov, width, height, t_far, out)
        return out

    def probe_rays(self, g: Grid, count, seed) -> np.ndarray:
        out = np.zeros((count, 8), np.float64)
        self.L.ref_probe_rays(np.asarray(g.res, np.int32), np.asarray(g.wmin, np.float64),
                              g.voxel, count, seed, out)
        return out

    def random_rays(self, g: Grid, count, seed) -> np.ndarray:
        out = np.zeros((count, 8), np.float64)
        self.L.ref_random_rays(np.asarray(g.res, np.int32), np.asarray(g.wmin, np.float64),
                               g.voxel, count, seed, out)
        return out

    def random_grid(self, res, wmin, voxel, seed, fraction) -> Grid:
        r = np.asarray(res, np.int32)
        bits = np.zeros(self._nbytes(r), np.uint8)
        self.L.ref_random_grid(r, np.asarray(wmin, np.float64), voxel, seed, fraction, bits)
        return Grid(tuple(int(x) for x in r), tuple(wmin), voxel, bits)

    def random_blocky_grid(self, res, wmin, voxel, seed, block_fraction, noise) -> Grid:
        r = np.asarray(res, np.int32)
        bits = np.zeros(self._nbytes(r), np.uint8)
        self.L.ref_random_blocky_grid(r, np.asarray(wmin, np.float64), voxel, seed,
                                      block_fraction, noise, bits)
        return Grid(tuple(int(x) for x in r), tuple(wmin), voxel, bits)

    def sog1(self, g: Grid) -> bytes:
        args = (np.asarray(g.res, np.int32), np.asarray(g.wmin, np.float64), g.voxel,
                np.ascontiguousarray(g.bits))
        n = self.L.ref_build_sog1(*args, None, 0)
        buf = (C.c_uint8 * n)()
        self.L.ref_build_sog1(*args, buf, n)
        return bytes(buf)

    def sampler(self, levels, analyzer, kernel, sched_kind, dt0, growth=0.0, cascade=False):
        res = np.asarray(levels[0].res, np.int32)
        wm = np.concatenate([np.asarray(g.wmin, np.float64) for g in levels])
        vx = np.asarray([g.voxel for g in levels], np.float64)
        keep = [np.ascontiguousarray(g.bits) for g in levels]
        ptrs = (C.c_void_p * len(levels))(*[k.ctypes.data for k in keep])
        h = self.L.ref_sampler_create(len(levels), 1 if cascade else 0, res, wm, vx, ptrs,
                                      analyzer, kernel, sched_kind, dt0, growth)
        return _RefSampler(self, h, keep)


class _RefSampler:
    def __init__(self, lib: RefLib, h, keep):
        self.lib, self.h, self._keep = lib, h, keep

    def __del__(self):
        try:
            self.lib.L.ref_sampler_free(self.h)
        except Exception:
            pass

    def sample(self, rays: np.ndarray, skip: np.ndarray | None = None, threads: int = 0) -> Packed:
        rays = np.ascontiguousarray(rays, np.float64).reshape(-1, 8)
        n = rays.shape[0]
        threads = threads or max(1, os.cpu_count() or 1)
        sk = None if skip is None else np.ascontiguousarray(skip, np.uint8)
        skp = None if sk is None else sk.ctypes.data
        cap = max(1024, 64 * n)
        while True:
            pi = np.zeros((n, 2), np.int64)
            ts = np.zeros(cap, np.float64)
            te = np.zeros(cap, np.float64)
            ce = np.zeros(cap, np.uint32)
            lv = np.zeros(cap, np.uint8)
            ct = np.zeros((n, 3), np.int32)
            tot = self.lib.L.ref_sample_batch(self.h, rays, n, skp, threads, cap, pi, ts, te, ce,
                                              lv, ct)
            if tot <= cap:
                ri = np.repeat(np.arange(n, dtype=np.int32), pi[:, 1])
                st = np.zeros(n, np.uint8) if sk is None else (sk != 0).astype(np.uint8) * 2
                return Packed(pi, ts[:tot], te[:tot], ri, ce[:tot], lv[:tot], ct, st)
            cap = int(tot)

    def events(self, ray, cap: int = 1 << 16):
        ev = np.zeros((cap, 6), np.int32)
        tt = np.zeros((cap, 2), np.float64)
        ctr = np.zeros(2, np.int64)
        n = self.lib.L.ref_collect_events(self.h, np.ascontiguousarray(ray, np.float64), cap, ev,
                                          tt, ctr)
        out = [(tuple(int(v) for v in ev[i, :3]), int(ev[i, 3]), float(tt[i, 0]), float(tt[i, 1]),
                int(ev[i, 4]), int(ev[i, 5])) for i in range(min(n, cap))]
        return n, out, ctr

    def time(self, rays: np.ndarray, skip=None, threads: int = 0, reps: int = 1):
        rays = np.ascontiguousarray(rays, np.float64).reshape(-1, 8)
        threads = threads or max(1, os.cpu_count() or 1)
        sk = None if skip is None else np.ascontiguousarray(skip, np.uint8)
        samples = C.c_int64(0)
        sec = self.lib.L.ref_time_sampler(self.h, rays, rays.shape[0],
                                          None if sk is None else sk.ctypes.data, threads, reps,
                                          C.byref(samples))
        return sec, samples.value
