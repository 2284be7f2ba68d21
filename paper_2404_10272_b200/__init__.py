"""paper_2404_10272_b200 — B200-native VDB/HDDA ray sampler (arXiv 2404.10272 hot path).

Python host mirror of the reference's C++ API (namespace ``sog``) over the C-ABI
in ``include/sogk.h`` (``_lib/libsogk.so``, sm_100a).  Names, argument meaning
and error behaviour follow the reference:

===========================  ==========================================================
reference (``sog::``)         here
===========================  ==========================================================
GridTransform (grid.hpp:18)   ``GridTransform``
DenseGrid (grid.hpp:120)      ``DenseGrid`` (HBM-resident bit payload)
build_sparse (sparse.hpp:333) ``build_sparse`` -> ``SparseGrid`` (GPU-built VDB)
serialize_* / deserialize_*   ``serialize_dense/sparse``, ``deserialize_dense/sparse``
  (io.hpp:134-214)
memory_bytes (io.hpp:223)     ``memory_bytes``
StepSchedule (sampling.hpp:18) ``StepSchedule.constant / .linear``
KernelKind (sampling.hpp:155) ``KernelKind.branch / .skip``
run_sampler (sampling.hpp:166) ``run_sampler`` (one ray, SampleRun)
run_cascade_sampler (:440)    ``run_cascade_sampler``
make_sampler (bench.hpp:382)  ``make_sampler`` -> batched ``Sampler``
Camera (camera.hpp:158)       ``Camera``
generate_scene, ...           ``generate_scene``, ``build_dense_cascade``,
  (scene_gen.hpp)               ``make_probe_rays``, ``random_rays`` ...
===========================  ==========================================================

Errors: ``std::invalid_argument`` -> ``ValueError``; ``sog::io_error`` -> ``IoError``
(with ``.code``); device failures -> ``RuntimeError``.  There is no CPU fallback:
every sampling call runs the CUDA kernels of libsogk.so and fails loudly when the
library or a GPU is missing.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "lib", "GridTransform", "DenseGrid", "SparseGrid", "build_sparse", "StepSchedule",
    "KernelKind", "Analyzer", "Sampler", "PackedSamples", "SampleRun", "run_sampler",
    "run_cascade_sampler", "make_sampler", "Camera", "generate_scene", "build_dense_cascade",
    "make_probe_rays", "random_rays", "random_grid", "random_blocky_grid", "serialize_dense",
    "serialize_sparse", "deserialize_dense", "deserialize_sparse", "memory_bytes", "IoError",
    "SceneKind", "RAY_OK", "RAY_INVALID", "RAY_UNDEFINED", "Traversal", "collect_events",
    "dump_trace", "query", "EVENT_DTYPE", "QUERY_DTYPE",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SOGK_LIB") or os.path.join(_HERE, "_lib", "libsogk.so")

OK, INVALID_ARG, CUDA_ERROR, OOM, INSUFFICIENT_CAPACITY, IO_ERROR, NO_DEVICE = range(7)
RAY_OK, RAY_INVALID, RAY_UNDEFINED = 0, 1, 2
STATS_LEN = 8
(STAT_TOTAL_SAMPLES, STAT_INVALID_RAYS, STAT_UNDEFINED_RAYS, STAT_ANALYZER_LOOKUPS,
 STAT_ANALYZER_STEPS, STAT_KERNEL_LOOKUPS, STAT_SLAB_OVERFLOW_RAYS) = range(7)


# sogk_event = sog::TraversalEvent / CascadeEvent (grid.hpp:98-104, sampling.hpp:297-299)
EVENT_DTYPE = np.dtype([("ijk", np.int32, 3), ("level", np.int32), ("t0", np.float64), ("t1", np.float64),
                        ("occupied", np.int32), ("grid_level", np.int32)])
# sogk_query = sog::QueryResult (sparse.hpp:130-135)
QUERY_DTYPE = np.dtype([("occupied", np.int32), ("level", np.int32), ("origin", np.int32, 3),
                        ("extent", np.int32)])
LEVEL_NAMES = ("leaf_voxel", "leaf_tile", "internal_tile", "root_tile")  # level_name (grid.hpp:84-91)


class IoError(RuntimeError):
    """sog::io_error (io.hpp:17-36): ``code`` is one of bad magic / bad version / truncated / corrupt."""

    def __init__(self, msg: str):
        super().__init__(msg)
        self.code = next((c for c in ("bad magic", "bad version", "truncated", "corrupt")
                          if c in msg), "corrupt")


class _Transform(C.Structure):
    _fields_ = [("res", C.c_int32 * 3), ("world_min", C.c_double * 3), ("voxel_size", C.c_double)]


class _GridInfo(C.Structure):
    _fields_ = [("kind", C.c_int32), ("transform", _Transform), ("root_entries", C.c_int64),
                ("internal_nodes", C.c_int64), ("leaf_count", C.c_int64),
                ("memory_bytes", C.c_int64), ("device_bytes", C.c_int64)]


class _SamplerDesc(C.Structure):
    _fields_ = [("analyzer", C.c_int32), ("kernel", C.c_int32), ("schedule", C.c_int32),
                ("dt0", C.c_double), ("growth", C.c_double), ("cascade", C.c_int32),
                ("spin_cap", C.c_int32)]


class _Camera(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("forward", C.c_double * 3),
                ("right", C.c_double * 3), ("cam_up", C.c_double * 3), ("tan_half", C.c_double),
                ("aspect", C.c_double), ("t_far", C.c_double), ("width", C.c_int32),
                ("height", C.c_int32)]


class _Primitive(C.Structure):  # sogk_primitive = sog::Primitive (render.hpp:19-56)
    _fields_ = [("shape", C.c_int32), ("center", C.c_double * 3), ("radius", C.c_double),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("density", C.c_double),
                ("color", C.c_double * 3)]


_vp, _i64, _i32, _dbl, _u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_uint64
_SIGS = {
    "sogk_version": (C.c_char_p, []),
    "sogk_abi_version": (C.c_int, []),
    "sogk_status_string": (C.c_char_p, [C.c_int]),
    "sogk_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
    "sogk_device_count": (C.c_int, []),
    "sogk_grid_create_dense": (C.c_int, [C.POINTER(_Transform), _vp, C.c_size_t, _vp, C.POINTER(_vp)]),
    "sogk_grid_create_dense_device": (C.c_int, [C.POINTER(_Transform), _vp, C.c_size_t, _vp, C.POINTER(_vp)]),
    "sogk_grid_build_vdb": (C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    "sogk_grid_build_distance": (C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    "sogk_grid_download_distance": (C.c_int, [_vp, _vp, C.c_size_t, C.POINTER(_i32)]),
    "sogk_grid_load_sog0": (C.c_int, [_vp, C.c_size_t, _vp, C.POINTER(_vp)]),
    "sogk_grid_load_sog1": (C.c_int, [_vp, C.c_size_t, _vp, C.POINTER(_vp)]),
    "sogk_grid_export_sog0": (C.c_int, [_vp, _vp, C.POINTER(C.c_size_t)]),
    "sogk_grid_export_sog1": (C.c_int, [_vp, _vp, C.POINTER(C.c_size_t)]),
    "sogk_grid_download_dense": (C.c_int, [_vp, _vp, C.c_size_t]),
    "sogk_grid_get_info": (C.c_int, [_vp, C.POINTER(_GridInfo)]),
    "sogk_grid_destroy": (C.c_int, [_vp]),
    "sogk_sampler_create": (C.c_int, [C.POINTER(_vp), C.c_int, C.POINTER(_SamplerDesc), C.POINTER(_vp)]),
    "sogk_sampler_destroy": (C.c_int, [_vp]),
    "sogk_sampler_set_ray_order": (C.c_int, [_vp, C.c_int]),
    "sogk_release_workspaces": (C.c_int, []),
    "sogk_sample_count": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "sogk_sample_write": (C.c_int, [_vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sogk_sample_count_ex": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, C.POINTER(_u64)]),
    "sogk_sample_write_ex": (C.c_int, [_vp, _vp, _i64, _vp, _u64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sogk_sample_count_camera": (C.c_int, [_vp, C.POINTER(_Camera), _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "sogk_sample_write_camera": (C.c_int, [_vp, C.POINTER(_Camera), _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sogk_sample_host": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sogk_traverse_count": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "sogk_traverse_write": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _vp]),
    "sogk_traverse_host": (C.c_int, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sogk_grid_query": (C.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "sogk_grid_query_host": (C.c_int, [_vp, _vp, _i64, _vp]),
    "sogk_camera_setup": (C.c_int, [_vp, _vp, _vp, _dbl, _i32, _i32, _dbl, C.POINTER(_Camera)]),
    "sogk_camera_rays": (C.c_int, [C.POINTER(_Camera), _i64, _i64, _vp, _vp]),
    "sogk_camera_rays_host": (C.c_int, [C.POINTER(_Camera), _i64, _i64, _vp]),
    "sogk_scene_analytic": (C.c_int, [C.c_int, C.POINTER(_Transform), _u64, _i32, _vp, _i32, C.POINTER(_i32), _vp]),
    "sogk_scene_create": (C.c_int, [_vp, _i32, _vp, C.POINTER(_vp)]),
    "sogk_scene_destroy": (C.c_int, [_vp]),
    "sogk_composite": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "sogk_render_camera": (C.c_int, [_vp, _vp, C.POINTER(_Camera), _i64, _i64, _vp, _vp, _vp, _vp]),
    "sogk_render_frame_host": (C.c_int, [_vp, _vp, C.POINTER(_Camera), _vp, _vp, _vp]),
    "sogk_scene_generate": (C.c_int, [C.c_int, C.POINTER(_Transform), _u64, _dbl, _i32, _dbl, _vp, C.POINTER(_dbl)]),
    "sogk_scene_cascade": (C.c_int, [C.c_int, C.POINTER(_Transform), _u64, _dbl, _i32, _dbl, _i32, _vp, C.POINTER(_Transform)]),
    "sogk_probe_rays": (C.c_int, [C.POINTER(_Transform), _i64, _u64, _vp]),
    "sogk_random_rays": (C.c_int, [C.POINTER(_Transform), _i64, _u64, _vp]),
    "sogk_random_grid": (C.c_int, [C.POINTER(_Transform), _u64, _dbl, _vp]),
    "sogk_random_blocky_grid": (C.c_int, [C.POINTER(_Transform), _u64, _dbl, _dbl, _vp]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    return L


lib = _load()


def _last_error() -> str:
    buf = C.create_string_buffer(1024)
    lib.sogk_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def _check(status: int, what: str = ""):
    if status == OK:
        return
    msg = f"{what}: {_last_error()}" if what else _last_error()
    if status == INVALID_ARG:
        raise ValueError(msg)
    if status == IO_ERROR:
        raise IoError(msg)
    if status == OOM:
        raise MemoryError(msg)
    raise RuntimeError(f"{lib.sogk_status_string(status).decode()}: {msg}")


def _ptr(x) -> Optional[int]:
    """Raw address of a torch tensor / numpy array (None passes NULL)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


def _stream(stream) -> Optional[int]:
    if stream is None:
        try:
            import torch

            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream or None
        except Exception:  # pragma: no cover
            return None
        return None
    return getattr(stream, "cuda_stream", stream) or None


# ---------------------------------------------------------------------------
# grids
# ---------------------------------------------------------------------------
class SceneKind:
    blobs, shell, sponge, random = 0, 1, 2, 3
    names = {"blobs": 0, "shell": 1, "sponge": 2, "random": 3}


@dataclass(frozen=True)
class GridTransform:
    """sog::GridTransform (grid.hpp:18-70)."""

    resolution: tuple = (1, 1, 1)
    world_min: tuple = (0.0, 0.0, 0.0)
    voxel_size: float = 1.0

    def __post_init__(self):
        r = tuple(int(x) for x in self.resolution)
        object.__setattr__(self, "resolution", r)
        object.__setattr__(self, "world_min", tuple(float(x) for x in self.world_min))
        if min(r) < 1:
            raise ValueError("grid resolution components must be >= 1")
        if not self.voxel_size > 0.0:
            raise ValueError("voxel size must be positive")

    @staticmethod
    def cube(res: int, wmin=(0.0, 0.0, 0.0), extent: float = 1.0) -> "GridTransform":
        return GridTransform((res, res, res), wmin, extent / res)

    def world_max(self):
        return tuple(self.world_min[a] + self.resolution[a] * self.voxel_size for a in range(3))

    def voxel_count(self) -> int:
        return self.resolution[0] * self.resolution[1] * self.resolution[2]

    def payload_bytes(self) -> int:
        return (self.voxel_count() + 7) // 8

    def _c(self) -> _Transform:
        t = _Transform()
        for a in range(3):
            t.res[a] = self.resolution[a]
            t.world_min[a] = self.world_min[a]
        t.voxel_size = self.voxel_size
        return t

    @staticmethod
    def _from_c(t: _Transform) -> "GridTransform":
        return GridTransform(tuple(t.res), tuple(t.world_min), t.voxel_size)


class _Grid:
    _kind = -1

    def __init__(self, handle: int, transform: GridTransform):
        self._h = handle
        self.transform_ = transform

    def transform(self) -> GridTransform:
        return self.transform_

    def info(self) -> _GridInfo:
        inf = _GridInfo()
        _check(lib.sogk_grid_get_info(self._h, C.byref(inf)), "grid info")
        return inf

    def payload(self) -> np.ndarray:
        """DenseGrid::payload() (a VDB is expanded like to_dense, sparse.hpp:374-383)."""
        out = np.zeros(self.transform_.payload_bytes(), np.uint8)
        _check(lib.sogk_grid_download_dense(self._h, _ptr(out), out.size), "download")
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib.sogk_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DenseGrid(_Grid):
    """sog::DenseGrid (grid.hpp:120-165), payload resident in HBM."""

    _kind = 0

    def __init__(self, transform: GridTransform, bits=None, stream=None, _handle=None):
        if _handle is not None:
            super().__init__(_handle, transform)
            return
        if bits is None:
            bits = np.zeros(transform.payload_bytes(), np.uint8)
        h = C.c_void_p()
        tc = transform._c()
        if hasattr(bits, "is_cuda") and bits.is_cuda:
            st = lib.sogk_grid_create_dense_device(C.byref(tc), bits.data_ptr(), bits.numel(),
                                                   _stream(stream), C.byref(h))
        else:
            b = np.ascontiguousarray(np.asarray(bits, np.uint8))
            st = lib.sogk_grid_create_dense(C.byref(tc), _ptr(b), b.size, _stream(stream),
                                            C.byref(h))
        _check(st, "DenseGrid")
        super().__init__(h.value, transform)

    def memory_bytes(self) -> int:
        return self.transform_.payload_bytes()


class SparseGrid(_Grid):
    """sog::SparseGrid (sparse.hpp:141-218) as the GPU VDB layout (csrc/sogk_layout.h)."""

    _kind = 1

    def leaf_count(self) -> int:
        return int(self.info().leaf_count)

    def root_size(self) -> int:
        return int(self.info().root_entries)

    def memory_bytes(self) -> int:
        return int(self.info().memory_bytes)


def build_sparse(dense: DenseGrid, stream=None) -> SparseGrid:
    """build_sparse (sparse.hpp:333-371) on the GPU (K1, csrc/sogk_vdb.cu)."""
    if not isinstance(dense, DenseGrid):
        raise ValueError("build_sparse needs a DenseGrid")
    h = C.c_void_p()
    _check(lib.sogk_grid_build_vdb(dense._h, _stream(stream), C.byref(h)), "build_sparse")
    return SparseGrid(h.value, dense.transform())


class DistanceGrid(_Grid):
    """sog::DistanceGrid (distance.hpp:15-43): chessboard distance per voxel, in HBM."""

    _kind = 2

    def distances(self) -> np.ndarray:
        """int32 [z][y][x] (the payload DistanceGrid::at reads in bounds)."""
        t = self.transform()
        out = np.empty(t.voxel_count(), np.int32)
        _check(lib.sogk_grid_download_distance(self._h, _ptr(out), out.size, None), "distance")
        return out.reshape(t.resolution[2], t.resolution[1], t.resolution[0])

    def all_empty(self) -> bool:
        ae = C.c_int32(0)
        _check(lib.sogk_grid_download_distance(self._h, None, 0, C.byref(ae)), "distance")
        return bool(ae.value)

    def memory_bytes(self) -> int:
        return int(self.info().memory_bytes)


def build_distance(dense: DenseGrid, stream=None) -> DistanceGrid:
    """build_distance (distance.hpp:45-103) on the GPU (exact separable transform)."""
    if not isinstance(dense, DenseGrid):
        raise ValueError("build_distance needs a DenseGrid")
    h = C.c_void_p()
    _check(lib.sogk_grid_build_distance(dense._h, _stream(stream), C.byref(h)), "build_distance")
    return DistanceGrid(h.value, dense.transform())


def _export(fn, h) -> bytes:
    n = C.c_size_t(0)
    _check(fn(h, None, C.byref(n)), "export")
    buf = (C.c_uint8 * n.value)()
    _check(fn(h, buf, C.byref(n)), "export")
    return bytes(buf)


def serialize_dense(g: DenseGrid) -> bytes:
    return _export(lib.sogk_grid_export_sog0, g._h)


def serialize_sparse(g: SparseGrid) -> bytes:
    return _export(lib.sogk_grid_export_sog1, g._h)


def deserialize_dense(data: bytes) -> DenseGrid:
    h = C.c_void_p()
    b = np.frombuffer(bytes(data), np.uint8)
    _check(lib.sogk_grid_load_sog0(_ptr(b) if b.size else None, b.size, None, C.byref(h)),
           "deserialize_dense")
    inf = _GridInfo()
    _check(lib.sogk_grid_get_info(h, C.byref(inf)))
    return DenseGrid(GridTransform._from_c(inf.transform), _handle=h.value)


def deserialize_sparse(data: bytes) -> SparseGrid:
    h = C.c_void_p()
    b = np.frombuffer(bytes(data), np.uint8)
    _check(lib.sogk_grid_load_sog1(_ptr(b) if b.size else None, b.size, None, C.byref(h)),
           "deserialize_sparse")
    inf = _GridInfo()
    _check(lib.sogk_grid_get_info(h, C.byref(inf)))
    return SparseGrid(h.value, GridTransform._from_c(inf.transform))


def memory_bytes(g: _Grid) -> int:
    """sog::memory_bytes (io.hpp:223-238)."""
    return g.memory_bytes()


# ---------------------------------------------------------------------------
# schedules, kernels, samplers
# ---------------------------------------------------------------------------
class KernelKind:
    branch, skip = 0, 1


class Analyzer:
    dda, hdda, cd = 0, 1, 2


@dataclass(frozen=True)
class StepSchedule:
    """sog::StepSchedule (sampling.hpp:18-39)."""

    kind: int = 0  # 0 constant, 1 linear
    dt0: float = 1.0
    growth: float = 0.0

    @staticmethod
    def constant(dt: float) -> "StepSchedule":
        if not dt > 0.0:
            raise ValueError("step size must be positive")
        return StepSchedule(0, float(dt), 0.0)

    @staticmethod
    def linear(dt0: float, growth: float = 1.0 / 256.0) -> "StepSchedule":
        if not dt0 > 0.0:
            raise ValueError("step size must be positive")
        if growth < 0.0:
            raise ValueError("growth must be non-negative")
        return StepSchedule(1, float(dt0), float(growth))

    def step(self, t: float) -> float:
        return self.dt0 if self.kind == 0 else max(self.dt0, self.growth * t)


@dataclass
class PackedSamples:
    """Packed intervals of a ray batch (include/sogk.h output contract)."""

    packed_info: object  # [n, 2] int64 (offset, count)
    t_starts: object
    t_ends: object
    ray_indices: object
    cells: object
    levels: object
    status: object = None
    counters: object = None
    stats: Optional[np.ndarray] = None

    @property
    def total(self) -> int:
        return int(self.stats[STAT_TOTAL_SAMPLES]) if self.stats is not None else len(self.t_starts)


@dataclass
class SampleRun:
    """sog::SampleRun (sampling.hpp:157-164)."""

    samples: list = field(default_factory=list)
    analyzer_lookups: int = 0
    analyzer_steps: int = 0
    kernel_lookups: int = 0
    t_ends: list = field(default_factory=list)
    cells: list = field(default_factory=list)
    levels: list = field(default_factory=list)
    status: int = RAY_OK

    def total_lookups(self) -> int:
        return self.analyzer_lookups + self.kernel_lookups


class _nullctx:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("sampling needs a CUDA device (there is no CPU fallback)")
    return torch


class Sampler:
    """One sampler variant over one grid or a cascade (make_sampler, bench.hpp:382-413).

    The batched two-pass API works on torch CUDA tensors (device buffers):
    ``count(rays) -> (packed_info, stats)`` then ``write(rays, packed_info, total)``.
    """

    def __init__(self, levels: Sequence[_Grid], analyzer: int, kernel: int,
                 schedule: StepSchedule, cascade: bool = False, spin_cap: int = 0,
                 ray_order: int = 0):
        levels = list(levels)
        self.levels = levels  # keep the grids alive
        self.analyzer, self.kernel, self.schedule = analyzer, kernel, schedule
        arr = (C.c_void_p * max(1, len(levels)))(*[g._h for g in levels])
        d = _SamplerDesc(analyzer, kernel, schedule.kind, schedule.dt0, schedule.growth,
                         1 if cascade else 0, spin_cap)
        h = C.c_void_p()
        _check(lib.sogk_sampler_create(arr, len(levels), C.byref(d), C.byref(h)), "sampler")
        self._h = h.value
        self._tokens = {}
        if ray_order:  # pass 1 in binned order (incoherent rays); outputs unchanged
            _check(lib.sogk_sampler_set_ray_order(self._h, ray_order), "ray order")

    def __del__(self):
        try:
            if self._h:
                lib.sogk_sampler_destroy(self._h)
                self._h = None
        except Exception:
            pass

    # -- device two-pass API ------------------------------------------------
    # count() keeps the handshake token of its run slabs per packed_info buffer
    # (sogk_sample_count_ex); write() presents the token of the count that last filled its
    # packed_info, and the library uses the slabs only if that count is still the latest on the
    # write's stream -- a write can never pick up another count's slabs (it takes the exact cold
    # path instead), whatever happened to the ray buffer in between
    def count(self, rays, status=None, counters=None, stream=None, packed_info=None, stats=None):
        torch = _torch()
        n = rays.shape[0]
        dev = rays.device
        packed = packed_info if packed_info is not None else torch.empty((n, 2), dtype=torch.int64, device=dev)
        st = stats if stats is not None else torch.empty(STATS_LEN, dtype=torch.int64, device=dev)
        tok = _u64(0)
        sh = _stream(stream)
        _check(lib.sogk_sample_count_ex(self._h, _ptr(rays), n, _ptr(packed), _ptr(st), _ptr(status),
                                        _ptr(counters), sh, C.byref(tok)), "sample_count")
        key = _ptr(packed)
        self._tokens.pop(key, None)
        self._tokens[key] = (tok.value, _ptr(rays), n)
        while len(self._tokens) > 64:  # only the latest counts can still own a workspace
            self._tokens.pop(next(iter(self._tokens)))
        return packed, st

    def write(self, rays, packed_info, total: int, ray_index_base: int = 0, stream=None,
              out: Optional[dict] = None, cells: bool = True, levels: bool = True):
        torch = _torch()
        dev = rays.device
        o = out or {}

        def buf(key, dtype):  # the caller's buffer, or a new one (allocated only when missing)
            return o[key] if key in o else torch.empty(total, dtype=dtype, device=dev)

        ts = buf("t_starts", torch.float64)
        te = buf("t_ends", torch.float64)
        ri = buf("ray_indices", torch.int32)
        ce = buf("cells", torch.int32) if cells else None
        lv = buf("levels", torch.uint8) if levels else None
        if total == 0:  # nothing to write (empty tensors have no device address)
            return ts, te, ri, ce, lv
        sh = _stream(stream)
        n = rays.shape[0]
        tok, rp, tn = self._tokens.get(_ptr(packed_info), (0, None, -1))
        if (rp, tn) != (_ptr(rays), n):
            tok = 0  # packed_info was not filled by a count of these rays: exact cold path
        _check(lib.sogk_sample_write_ex(self._h, _ptr(rays), n, _ptr(packed_info), tok,
                                        ray_index_base, _ptr(ts), _ptr(te), _ptr(ri), _ptr(ce),
                                        _ptr(lv), sh), "sample_write")
        return ts, te, ri, ce, lv

    def count_camera(self, cam: "Camera", first: int, n: int, packed_info, stats, stream=None,
                     status=None, counters=None):
        c = cam._c()
        _check(lib.sogk_sample_count_camera(self._h, C.byref(c), first, n, _ptr(packed_info),
                                            _ptr(stats), _ptr(status), _ptr(counters),
                                            _stream(stream)), "sample_count_camera")

    def write_camera(self, cam: "Camera", first: int, n: int, packed_info, ts, te=None, ri=None,
                     ce=None, lv=None, ray_index_base: int = 0, stream=None):
        c = cam._c()
        _check(lib.sogk_sample_write_camera(self._h, C.byref(c), first, n, _ptr(packed_info),
                                            ray_index_base, _ptr(ts), _ptr(te), _ptr(ri), _ptr(ce),
                                            _ptr(lv), _stream(stream)), "sample_write_camera")

    def sample(self, rays, ray_index_base: int = 0, stream=None, with_counters: bool = True) -> PackedSamples:
        """Both passes on device rays (torch CUDA tensor [n, 8] float64).  With `stream`, the
        outputs are allocated on it and the total is read back in its order."""
        torch = _torch()
        if stream is not None and not isinstance(stream, torch.cuda.Stream):
            stream = torch.cuda.ExternalStream(int(_stream(stream)))
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            n = rays.shape[0]
            status = torch.empty(n, dtype=torch.uint8, device=rays.device)
            counters = torch.empty((n, 3), dtype=torch.int32, device=rays.device) if with_counters else None
            packed, stats = self.count(rays, status, counters, stream)
            hs = stats.cpu().numpy()  # on `stream` (the current stream here)
            total = int(hs[STAT_TOTAL_SAMPLES])
            ts, te, ri, ce, lv = self.write(rays, packed, total, ray_index_base, stream)
        if stream is not None:  # outputs usable in the caller's stream order
            torch.cuda.current_stream().wait_stream(stream)
        return PackedSamples(packed, ts, te, ri, ce, lv, status, counters, hs)

    # -- traverse (the analyzers' event streams) ----------------------------
    def traverse(self, rays, stream=None) -> "Traversal":
        """collect_events of every ray on the device (sogk_traverse_count / _write): torch
        tensors event_info [n, 2] (offset, count), events (uint8 [total, 40], view with
        EVENT_DTYPE), status, counters [n, 2] (lookup_count, step_count)."""
        torch = _torch()
        n = rays.shape[0]
        dev = rays.device
        info = torch.empty((n, 2), dtype=torch.int64, device=dev)
        stats = torch.zeros(STATS_LEN, dtype=torch.int64, device=dev)
        status = torch.empty(n, dtype=torch.uint8, device=dev)
        counters = torch.empty((n, 2), dtype=torch.int32, device=dev)
        sh = _stream(stream)
        _check(lib.sogk_traverse_count(self._h, _ptr(rays), n, _ptr(info), _ptr(stats), _ptr(status),
                                       _ptr(counters), sh), "traverse_count")
        with torch.cuda.stream(torch.cuda.ExternalStream(sh)) if sh else _nullctx():
            hs = stats.cpu().numpy()
        total = int(hs[STAT_TOTAL_SAMPLES])
        events = torch.empty((max(total, 1), EVENT_DTYPE.itemsize), dtype=torch.uint8, device=dev)
        if total:
            _check(lib.sogk_traverse_write(self._h, _ptr(rays), n, _ptr(info), _ptr(events), sh),
                   "traverse_write")
        return Traversal(info, events[:total], status, counters, hs)

    def traverse_host(self, rays: np.ndarray, stream=None) -> "Traversal":
        """The same from host rays (sogk_traverse_host): numpy outputs, events as EVENT_DTYPE."""
        rays = np.ascontiguousarray(rays, np.float64).reshape(-1, 8)
        n = rays.shape[0]
        cap = max(64, 64 * n)
        while True:
            info = np.zeros((n, 2), np.int64)
            ev = np.zeros(cap, EVENT_DTYPE)
            st = np.zeros(n, np.uint8)
            ct = np.zeros((n, 2), np.int32)
            stats = np.zeros(STATS_LEN, np.int64)
            rc = lib.sogk_traverse_host(self._h, _ptr(rays), n, cap, _ptr(info), ev.ctypes.data, _ptr(st),
                                        _ptr(ct), _ptr(stats), _stream(stream))
            if rc == INSUFFICIENT_CAPACITY:
                cap = int(stats[STAT_TOTAL_SAMPLES])
                continue
            _check(rc, "traverse_host")
            return Traversal(info, ev[:int(stats[STAT_TOTAL_SAMPLES])], st, ct, stats)

    # -- host end-to-end API ------------------------------------------------
    def sample_host(self, rays: np.ndarray, ray_index_base: int = 0, capacity: Optional[int] = None,
                    stream=None, out: Optional[dict] = None) -> PackedSamples:
        """sogk_sample_host: host rays in, host packed samples out (H2D/D2H inside)."""
        rays = np.ascontiguousarray(rays, np.float64).reshape(-1, 8)
        n = rays.shape[0]
        o = out or {}
        cap = capacity if capacity is not None else max(1024, 64 * n)
        while True:
            pi = o.get("packed_info", np.empty((n, 2), np.int64))
            ts = o.get("t_starts", np.empty(cap, np.float64))
            te = o.get("t_ends", np.empty(cap, np.float64))
            ri = o.get("ray_indices", np.empty(cap, np.int32))
            ce = o.get("cells", np.empty(cap, np.uint32))
            lv = o.get("levels", np.empty(cap, np.uint8))
            stt = o.get("status", np.empty(n, np.uint8))
            ct = o.get("counters", np.empty((n, 3), np.int32))
            stats = o.get("stats", np.zeros(STATS_LEN, np.int64))
            rc = lib.sogk_sample_host(self._h, _ptr(rays), n, ray_index_base, cap, _ptr(pi),
                                      _ptr(ts), _ptr(te), _ptr(ri), _ptr(ce), _ptr(lv), _ptr(stt),
                                      _ptr(ct), _ptr(stats), _stream(stream))
            if rc == INSUFFICIENT_CAPACITY and out is None:
                cap = int(stats[STAT_TOTAL_SAMPLES])
                continue
            _check(rc, "sample_host")
            tot = int(stats[STAT_TOTAL_SAMPLES])
            return PackedSamples(pi, ts[:tot], te[:tot], ri[:tot], ce[:tot], lv[:tot], stt, ct, stats)


@dataclass
class Traversal:
    """Event streams of a ray batch: ray r's events are events[info[r,0] : info[r,0] + info[r,1]];
    counters[r] = (lookup_count, step_count) after its last event (traversal.hpp:120-264)."""

    event_info: object
    events: object
    status: object
    counters: object
    stats: Optional[np.ndarray] = None

    def host_events(self) -> np.ndarray:
        ev = self.events
        if hasattr(ev, "cpu"):
            ev = ev.cpu().numpy()
        return np.ascontiguousarray(ev).reshape(-1).view(np.uint8).view(EVENT_DTYPE)

    def ray_events(self, r: int) -> np.ndarray:
        info = self.event_info.cpu().numpy() if hasattr(self.event_info, "cpu") else self.event_info
        o, c = info[r]
        return self.host_events()[o:o + c]


def dump_trace(events) -> str:
    """dump_trace (traversal.hpp:345-357): level, ijk, t0, t1 (%.17g), occupied per line."""
    out = []
    for e in events:
        i = e["ijk"]
        out.append(f"{LEVEL_NAMES[int(e['level'])]}\t{int(i[0])},{int(i[1])},{int(i[2])}\t"
                   f"{float(e['t0']):.17g}\t{float(e['t1']):.17g}\t{1 if e['occupied'] else 0}\n")
    return "".join(out)


def collect_events(grid_or_levels, ray, cascade: bool = False, spin_cap: int = 0):
    """collect_events(Analyzer(grid, ray)) (traversal.hpp:339-343) for one ray: DdaTraversal on a
    DenseGrid, HddaTraversal on a SparseGrid, CdTraversal on a DistanceGrid, CascadeTraversal on
    a list of levels -> (events [EVENT_DTYPE], lookup_count, step_count)."""
    levels = list(grid_or_levels) if isinstance(grid_or_levels, (list, tuple)) else [grid_or_levels]
    an = (Analyzer.hdda if isinstance(levels[0], SparseGrid) else
          Analyzer.cd if isinstance(levels[0], DistanceGrid) else Analyzer.dda)
    s = Sampler(levels, an, KernelKind.skip, StepSchedule.constant(1.0),
                cascade=cascade or len(levels) > 1, spin_cap=spin_cap)
    t = s.traverse_host(np.asarray(_ray_array(Ray.coerce(ray)), np.float64).reshape(1, 8))
    if int(t.status[0]) == RAY_UNDEFINED:
        raise RuntimeError("the reference analyzer never returns on this ray (edge-crossing spin)")
    if int(t.status[0]) == RAY_INVALID:
        raise ValueError("invalid ray")
    return t.events, int(t.counters[0, 0]), int(t.counters[0, 1])


def query(grid, ijk) -> np.ndarray:
    """SparseGrid::query (sparse.hpp:163-171) / DenseGrid::voxel_at for points int32 [n, 3]
    -> QUERY_DTYPE records (occupied, level, origin, extent)."""
    p = np.ascontiguousarray(np.asarray(ijk, np.int32).reshape(-1, 3))
    out = np.zeros(p.shape[0], QUERY_DTYPE)
    _check(lib.sogk_grid_query_host(grid._h, _ptr(p), p.shape[0], out.ctypes.data), "query")
    return out


def release_workspaces():
    """Free the pass-1 -> pass-2 workspaces (one per device and stream)."""
    _check(lib.sogk_release_workspaces(), "release_workspaces")


def make_sampler(grid_or_levels, analyzer: int, kernel: int, schedule: StepSchedule,
                 cascade: bool = False) -> Sampler:
    levels = grid_or_levels if isinstance(grid_or_levels, (list, tuple)) else [grid_or_levels]
    return Sampler(levels, analyzer, kernel, schedule, cascade)


def _single_ray(sampler: Sampler, ray) -> SampleRun:
    r = np.asarray(_ray_array(ray), np.float64).reshape(1, 8)
    p = sampler.sample_host(r)
    c = p.counters[0]
    return SampleRun(list(p.t_starts), int(c[0]), int(c[1]), int(c[2]), list(p.t_ends),
                     list(p.cells), list(p.levels), int(p.status[0]))


def _ray_array(ray):
    if isinstance(ray, Ray):
        return ray.as_array()
    return ray


def run_sampler(ray, grid: _Grid, kernel: int, sched: StepSchedule) -> SampleRun:
    """run_sampler (sampling.hpp:166-196): DDA on a DenseGrid, HDDA on a SparseGrid (slow: one ray)."""
    an = Analyzer.hdda if isinstance(grid, SparseGrid) else Analyzer.dda
    r = Ray.coerce(ray)
    return _single_ray(Sampler([grid], an, kernel, sched), r)


def run_cascade_sampler(ray, levels: Sequence[_Grid], kernel: int, sched: StepSchedule) -> SampleRun:
    """run_cascade_sampler (sampling.hpp:440-455)."""
    an = Analyzer.hdda if isinstance(levels[0], SparseGrid) else Analyzer.dda
    r = Ray.coerce(ray)
    return _single_ray(Sampler(list(levels), an, kernel, sched, cascade=True), r)


# ---------------------------------------------------------------------------
# rays, cameras, scenes (host generators in libsogk.so)
# ---------------------------------------------------------------------------
@dataclass
class Ray:
    """sog::Ray (ray.hpp:92-114) with the constructor's validation."""

    origin: tuple
    direction: tuple
    t_min: float = 0.0
    t_max: float = 1.7976931348623157e308

    def __post_init__(self):
        length = math.sqrt(self.direction[0] * self.direction[0] + self.direction[1] * self.direction[1]
                           + self.direction[2] * self.direction[2])
        if abs(length - 1.0) > 1e-9:
            raise ValueError("ray direction must be unit length")
        if not self.t_min >= 0.0:
            raise ValueError("ray t_min must be >= 0")
        if not self.t_min < self.t_max:
            raise ValueError("ray t_min must be < t_max")

    def as_array(self) -> np.ndarray:
        return np.array([*self.origin, *self.direction, self.t_min, self.t_max], np.float64)

    @staticmethod
    def coerce(r) -> "Ray":
        if isinstance(r, Ray):
            return r
        a = np.asarray(r, np.float64).reshape(8)
        return Ray(tuple(a[:3]), tuple(a[3:6]), float(a[6]), float(a[7]))


@dataclass
class Camera:
    """sog::Camera (camera.hpp:158-180)."""

    position: tuple = (0.0, 0.0, 2.0)
    target: tuple = (0.0, 0.0, 0.0)
    up: tuple = (0.0, 1.0, 0.0)
    vfov_deg: float = 45.0
    width: int = 160
    height: int = 120
    t_far: float = 1e6

    def _c(self) -> _Camera:
        c = _Camera()
        p = np.asarray(self.position, np.float64)
        t = np.asarray(self.target, np.float64)
        u = np.asarray(self.up, np.float64)
        _check(lib.sogk_camera_setup(_ptr(p), _ptr(t), _ptr(u), self.vfov_deg, self.width,
                                     self.height, self.t_far, C.byref(c)), "camera")
        return c

    def rays(self, first: int = 0, n: Optional[int] = None) -> np.ndarray:
        """Camera::pixel_ray for pixels [first, first+n), row-major, on the host."""
        n = self.width * self.height - first if n is None else n
        out = np.empty((n, 8), np.float64)
        c = self._c()
        _check(lib.sogk_camera_rays_host(C.byref(c), first, n, _ptr(out)), "camera rays")
        return out

    def rays_device(self, first: int = 0, n: Optional[int] = None, out=None, stream=None):
        """Same rays generated by the raygen kernel into a CUDA tensor."""
        torch = _torch()
        n = self.width * self.height - first if n is None else n
        out = out if out is not None else torch.empty((n, 8), dtype=torch.float64, device="cuda")
        c = self._c()
        _check(lib.sogk_camera_rays(C.byref(c), first, n, _ptr(out), _stream(stream)), "raygen")
        return out

    def pixel_ray(self, px: int, py: int) -> Ray:
        if px < 0 or py < 0 or px >= self.width or py >= self.height:
            raise IndexError("pixel outside image")  # std::out_of_range
        return Ray.coerce(self.rays(py * self.width + px, 1)[0])


def _kind(kind) -> int:
    return SceneKind.names[kind] if isinstance(kind, str) else int(kind)


def generate_scene(kind, transform: GridTransform, seed: int = 1, fraction: float = 0.05,
                   count: int = 12, threshold: float = 0.01):
    """generate_scene (scene_gen.hpp:94-192) -> (payload bits, occupancy)."""
    bits = np.zeros(transform.payload_bytes(), np.uint8)
    occ = C.c_double(0.0)
    tc = transform._c()
    _check(lib.sogk_scene_generate(_kind(kind), C.byref(tc), seed, fraction, count, threshold,
                                   _ptr(bits), C.byref(occ)), "generate_scene")
    return bits, occ.value


def build_dense_cascade(kind, base: GridTransform, levels: int, seed: int = 1,
                        fraction: float = 0.05, count: int = 12, threshold: float = 0.01):
    """build_dense_cascade(generate_scene(...).scene, base, levels) (scene_gen.hpp:196-209)
    -> list of (transform, bits)."""
    nb = base.payload_bytes()
    bits = np.zeros(nb * levels, np.uint8)
    ts = (_Transform * levels)()
    tc = base._c()
    _check(lib.sogk_scene_cascade(_kind(kind), C.byref(tc), seed, fraction, count, threshold,
                                  levels, _ptr(bits), ts), "build_dense_cascade")
    return [(GridTransform._from_c(ts[b]), bits[b * nb:(b + 1) * nb].copy()) for b in range(levels)]


def make_probe_rays(t: GridTransform, count: int, seed: int) -> np.ndarray:
    """make_probe_rays (bench.hpp:628-649) -> [count, 8] float64."""
    out = np.empty((count, 8), np.float64)
    tc = t._c()
    _check(lib.sogk_probe_rays(C.byref(tc), count, seed, _ptr(out)), "make_probe_rays")
    return out


def random_rays(t: GridTransform, count: int, seed: int) -> np.ndarray:
    """testsupport::random_ray x count from one mt19937_64(seed)."""
    out = np.empty((count, 8), np.float64)
    tc = t._c()
    _check(lib.sogk_random_rays(C.byref(tc), count, seed, _ptr(out)), "random_rays")
    return out


def random_grid(t: GridTransform, seed: int, fraction: float) -> np.ndarray:
    bits = np.zeros(t.payload_bytes(), np.uint8)
    tc = t._c()
    _check(lib.sogk_random_grid(C.byref(tc), seed, fraction, _ptr(bits)), "random_grid")
    return bits


def random_blocky_grid(t: GridTransform, seed: int, block_fraction: float,
                       noise_fraction: float) -> np.ndarray:
    bits = np.zeros(t.payload_bytes(), np.uint8)
    tc = t._c()
    _check(lib.sogk_random_blocky_grid(C.byref(tc), seed, block_fraction, noise_fraction,
                                       _ptr(bits)), "random_blocky_grid")
    return bits


# ---------------------------------------------------------------------------
# compositing consumer (render.hpp)
# ---------------------------------------------------------------------------
SPHERE, BOX = 0, 1


@dataclass
class Primitive:
    """sog::Primitive (render.hpp:19-56)."""

    shape: int = SPHERE
    center: tuple = (0.0, 0.0, 0.0)
    radius: float = 0.0
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (0.0, 0.0, 0.0)
    density: float = 0.0
    color: tuple = (1.0, 1.0, 1.0)

    @staticmethod
    def sphere(c, r, sigma, rgb) -> "Primitive":
        return Primitive(SPHERE, tuple(c), float(r), (0.0,) * 3, (0.0,) * 3, float(sigma), tuple(rgb))

    @staticmethod
    def box(lo, hi, sigma, rgb) -> "Primitive":
        return Primitive(BOX, (0.0,) * 3, 0.0, tuple(lo), tuple(hi), float(sigma), tuple(rgb))

    def _c(self) -> _Primitive:
        q = _Primitive()
        q.shape = self.shape
        q.radius = self.radius
        q.density = self.density
        for a in range(3):
            q.center[a], q.lo[a], q.hi[a], q.color[a] = self.center[a], self.lo[a], self.hi[a], self.color[a]
        return q


class AnalyticScene:
    """sog::AnalyticScene (render.hpp:58-92), uploaded to HBM (sogk_scene_create)."""

    def __init__(self, primitives: Sequence[Primitive] = (), background=(0.0, 0.0, 0.0)):
        self.primitives = list(primitives)
        self.background = tuple(float(x) for x in background)
        self._h = None

    @property
    def handle(self) -> int:
        """The HBM copy (AnalyticScene::validate + upload on first use)."""
        if self._h is None:
            arr = (_Primitive * max(1, len(self.primitives)))(*[p._c() for p in self.primitives])
            bg = np.asarray(self.background, np.float64)
            h = C.c_void_p()
            _check(lib.sogk_scene_create(C.cast(arr, C.c_void_p), len(self.primitives), _ptr(bg),
                                         C.byref(h)), "scene")
            self._h = h.value
        return self._h

    def __del__(self):
        try:
            if self._h:
                lib.sogk_scene_destroy(self._h)
                self._h = None
        except Exception:
            pass


def analytic_scene(kind, transform: GridTransform, seed: int = 1, count: int = 12) -> AnalyticScene:
    """generate_scene's AnalyticScene (scene_gen.hpp:94-176) on `transform`."""
    tc = transform._c()
    n = C.c_int32(0)
    _check(lib.sogk_scene_analytic(_kind(kind), C.byref(tc), seed, count, None, 0, C.byref(n), None),
           "scene_analytic")
    arr = (_Primitive * max(1, n.value))()
    bg = np.zeros(3, np.float64)
    _check(lib.sogk_scene_analytic(_kind(kind), C.byref(tc), seed, count, C.cast(arr, C.c_void_p),
                                   n.value, C.byref(n), _ptr(bg)), "scene_analytic")
    prims = [Primitive(q.shape, tuple(q.center), q.radius, tuple(q.lo), tuple(q.hi), q.density,
                       tuple(q.color)) for q in arr[:n.value]]
    return AnalyticScene(prims, tuple(bg))


@dataclass
class FrameResult:
    """render_frame's result (bench.hpp:415-421): image rows top to bottom, HxWx3 uint8."""

    image: np.ndarray
    lookups: int
    steps: int
    samples: int
    undefined: int = 0
    result: object = None  # [H*W, 5] color rgb, weight_sum, transmittance (device tensor)


def composite(sampler: "Sampler", scene: AnalyticScene, rays, packed_info, t_starts, stream=None):
    """composite_detailed (render.hpp:97-118) of every ray of a packed batch on the GPU:
    -> (result [n,5] = rgb, weight_sum, transmittance; rgb8 [n,3] = Image::set_pixel bytes)."""
    torch = _torch()
    n = rays.shape[0]
    res = torch.empty((n, 5), dtype=torch.float64, device=rays.device)
    rgb = torch.empty((n, 3), dtype=torch.uint8, device=rays.device)
    _check(lib.sogk_composite(sampler._h, scene.handle, _ptr(rays), n, _ptr(packed_info),
                              _ptr(t_starts) if t_starts.numel() else None, _ptr(res), _ptr(rgb),
                              _stream(stream)), "composite")
    return res, rgb


def render_frame(sampler: "Sampler", scene: AnalyticScene, camera: "Camera", stream=None) -> FrameResult:
    """render_frame (bench.hpp:424-461) as one fused sample + composite kernel per pixel."""
    torch = _torch()
    n = camera.width * camera.height
    res = torch.empty((n, 5), dtype=torch.float64, device="cuda")
    rgb = torch.empty((n, 3), dtype=torch.uint8, device="cuda")
    st = torch.zeros(STATS_LEN, dtype=torch.int64, device="cuda")
    c = camera._c()
    _check(lib.sogk_render_camera(sampler._h, scene.handle, C.byref(c), 0, n, _ptr(res), _ptr(rgb),
                                  _ptr(st), _stream(stream)), "render_camera")
    hs = st.cpu().numpy()
    img = rgb.cpu().numpy().reshape(camera.height, camera.width, 3)
    return FrameResult(img, int(hs[STAT_ANALYZER_LOOKUPS] + hs[STAT_KERNEL_LOOKUPS]),
                       int(hs[STAT_ANALYZER_STEPS]), int(hs[STAT_TOTAL_SAMPLES]),
                       int(hs[STAT_UNDEFINED_RAYS]), res)


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    """psnr (render.hpp:168-182) of two equally sized 8-bit images; 99 = identical."""
    if a.shape != b.shape:
        raise ValueError("psnr: image dimensions differ")
    d = a.astype(np.float64) - b.astype(np.float64)
    sq = float((d * d).sum())
    if sq == 0.0:
        return 99.0
    return min(99.0, 10.0 * math.log10(255.0 * 255.0 / (sq / d.size)))
