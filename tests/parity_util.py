"""Helpers shared by the parity tests: run the CUDA path through the C-ABI and
compare it bit-for-bit with the CPU oracle (oracle/sog_oracle.c)."""
from __future__ import annotations

import numpy as np

from oracle_bindings import BRANCH, CD, CONSTANT, DDA, HDDA, LINEAR, SKIP, Grid, Packed  # noqa: F401

VARIANTS = [(DDA, BRANCH), (DDA, SKIP), (HDDA, BRANCH), (HDDA, SKIP), (CD, BRANCH), (CD, SKIP)]


def host_grid(P, t, bits) -> Grid:
    return Grid(tuple(t.resolution), tuple(t.world_min), t.voxel_size, np.asarray(bits, np.uint8))


def scene_grid(P, kind, res=64, seed=1, fraction=0.05, count=12, wmin=(-1.0, -1.0, -1.0),
               extent=2.0) -> Grid:
    t = P.GridTransform.cube(res, wmin, extent)
    bits, _ = P.generate_scene(kind, t, seed=seed, fraction=fraction, count=count)
    return host_grid(P, t, bits)


def transform_of(P, g: Grid):
    return P.GridTransform(g.res, g.wmin, g.voxel)


def gpu_grids(P, levels, analyzer):
    dense = [P.DenseGrid(transform_of(P, g), g.bits) for g in levels]
    if analyzer == HDDA:
        return [P.build_sparse(d) for d in dense]
    if analyzer == CD:
        return [P.build_distance(d) for d in dense]
    return dense


def gpu_sample(P, levels, analyzer, kernel, sched, rays, cascade=False, ray_index_base=0,
               spin_cap=0) -> Packed:
    import torch

    grids = gpu_grids(P, levels, analyzer)
    s = P.Sampler(grids, analyzer, kernel, sched, cascade=cascade, spin_cap=spin_cap)
    d = torch.from_numpy(np.ascontiguousarray(rays, np.float64).reshape(-1, 8)).cuda()
    out = s.sample(d, ray_index_base=ray_index_base)
    torch.cuda.synchronize()
    return to_packed(out)


def to_packed(out) -> Packed:
    def np_(x):
        return None if x is None else (x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x))

    cells = np_(out.cells)
    return Packed(np_(out.packed_info), np_(out.t_starts), np_(out.t_ends), np_(out.ray_indices),
                  None if cells is None else cells.view(np.uint32), np_(out.levels),
                  np_(out.counters), np_(out.status))


def oracle_sample(oracle, levels, analyzer, kernel, sched, rays, cascade=False, ray_index_base=0):
    s = oracle.sampler(levels, analyzer, kernel, sched.kind, sched.dt0, sched.growth,
                       cascade=cascade)
    return oracle.sample(s, rays, ray_index_base)


def bits64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def assert_packed_equal(got: Packed, want: Packed, what: str = "", counters: bool = True,
                        cells: bool = True):
    n = want.packed_info.shape[0]
    assert got.packed_info.shape == (n, 2), what
    bad = np.nonzero((got.packed_info != want.packed_info).any(axis=1))[0]
    assert bad.size == 0, (f"{what}: packed_info differs on {bad.size} rays, first {bad[:5]}: "
                           f"got {got.packed_info[bad[:3]].tolist()} want {want.packed_info[bad[:3]].tolist()}")
    assert np.array_equal(got.status, want.status), f"{what}: status differs"
    assert np.array_equal(bits64(got.t_starts), bits64(want.t_starts)), f"{what}: t_starts differ"
    assert np.array_equal(bits64(got.t_ends), bits64(want.t_ends)), f"{what}: t_ends differ"
    assert np.array_equal(got.ray_indices, want.ray_indices), f"{what}: ray_indices differ"
    if cells:
        assert np.array_equal(got.cells, want.cells), f"{what}: cells differ"
        assert np.array_equal(got.levels, want.levels), f"{what}: levels differ"
    if counters:
        badc = np.nonzero((got.counters != want.counters).any(axis=1))[0]
        assert badc.size == 0, (f"{what}: counters differ on {badc.size} rays, first {badc[:5]}: "
                                f"got {got.counters[badc[:3]].tolist()} want {want.counters[badc[:3]].tolist()}")


def ref_sample(reflib, levels, analyzer, kernel, sched, rays, cascade=False, skip=None) -> Packed:
    """The unmodified reference (oracle/_ref: sog::run_sampler / run_cascade_sampler per ray on
    all host threads); rays with skip != 0 are not run (status 2, no samples)."""
    s = reflib.sampler(levels, analyzer, kernel, sched.kind, sched.dt0, sched.growth, cascade=cascade)
    return s.sample(rays, skip=skip)


def assert_rays_equal(got: Packed, want: Packed, mask, what: str = "", counters: bool = True,
                      cells: bool = True, ray_index_base: int = 0):
    """Per-ray comparison on the rays where mask is True (e.g. not spin-screened): counts,
    t_starts, t_ends, ray_indices, cells, levels (and counters) bit for bit."""
    mask = np.asarray(mask, bool)
    gc, wc = got.packed_info[:, 1], want.packed_info[:, 1]
    bad = np.nonzero(mask & (gc != wc))[0]
    assert bad.size == 0, f"{what}: counts differ on {bad.size} rays, first {bad[:5]}: {gc[bad[:3]]} vs {wc[bad[:3]]}"
    gsel = np.repeat(mask, gc)
    wsel = np.repeat(mask, wc)
    assert np.array_equal(bits64(got.t_starts)[gsel], bits64(want.t_starts)[wsel]), f"{what}: t_starts differ"
    assert np.array_equal(bits64(got.t_ends)[gsel], bits64(want.t_ends)[wsel]), f"{what}: t_ends differ"
    ri = np.repeat(np.arange(gc.size, dtype=np.int64) + ray_index_base, gc).astype(np.int32)
    assert np.array_equal(got.ray_indices, ri), f"{what}: ray_indices differ"
    if cells:
        assert np.array_equal(got.cells[gsel], want.cells[wsel]), f"{what}: cells differ"
        assert np.array_equal(got.levels[gsel], want.levels[wsel]), f"{what}: levels differ"
    if counters and want.counters is not None:
        badc = np.nonzero(mask & (got.counters != want.counters).any(axis=1))[0]
        assert badc.size == 0, f"{what}: counters differ on {badc.size} rays, first {badc[:5]}"
