"""Pass-2 expansion paths of gather_kernel (csrc/sogk_sample_kernels.cuh) against the oracle.

HDDA with the constant schedule expands batches that hold many long (tile) runs by output
position (gather_mp_batch): aligned outputs take two adjacent positions per thread with
2-wide stores, unaligned outputs one position per thread; batches of short runs keep the
per-run staged path.  These tests drive every branch -- long runs whose ladder crosses a
binade inside the run (the closed form's fallback), pairs that straddle run boundaries and
slab-overflow gaps (SOGK_SLAB=1: most of every ray comes from tail_kernel), and output
pointers that are not 16-byte aligned -- and require bit-exact output.
"""
import numpy as np
import pytest
import torch

from oracle_bindings import BRANCH, HDDA, SKIP
from parity_util import bits64, host_grid, oracle_sample

pytestmark = pytest.mark.gpu


def _tile_grid(P):
    """64^3 over [0, 1]^3: solid 16^3 blocks on the 8-voxel lattice (HDDA leaf tiles and
    collapsed nodes -> runs of tens of points) plus 1 % scattered voxels."""
    t = P.GridTransform.cube(64, (0.0, 0.0, 0.0), 1.0)
    rng = np.random.default_rng(5)
    occ = np.zeros((64, 64, 64), bool)  # [z, y, x]: x fastest, as the packed bits
    for _ in range(24):
        z, y, x = (rng.integers(0, 7, 3) * 8).tolist()
        occ[z:z + 16, y:y + 16, x:x + 16] = True
    occ |= rng.random(occ.shape) < 0.01
    return t, host_grid(P, t, np.packbits(occ.reshape(-1), bitorder="little"))


def _rays(P, t, n, seed):
    """Half random rays through the grid, half from x = -1.5 heading +x: t runs over
    [1.5, 2.5] inside the grid, so the ladder crosses the binade at t = 2 mid-tile."""
    rng = np.random.default_rng(seed)
    r = P.random_rays(t, n // 2, seed=seed)
    m = n - n // 2
    o = np.stack([np.full(m, -1.5), rng.uniform(0.02, 0.98, m), rng.uniform(0.02, 0.98, m)], 1)
    d = np.stack([np.ones(m), rng.uniform(-0.05, 0.05, m), rng.uniform(-0.05, 0.05, m)], 1)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    x = np.concatenate([o, d, np.zeros((m, 1)), np.full((m, 1), 10.0)], 1)
    return np.concatenate([np.asarray(r, np.float64).reshape(-1, 8), x], 0)


def _run(P, g, t, kernel, sched, rays, offset=0):
    """count + write through the C-ABI into buffers that start `offset` elements into a
    larger allocation (offset 1: 8-byte t arrays off the 16-byte boundary)."""
    s = P.Sampler([P.build_sparse(P.DenseGrid(t, g.bits))], HDDA, kernel, sched)
    d = torch.from_numpy(rays).cuda()
    packed, st = s.count(d)
    total = int(st.cpu()[P.STAT_TOTAL_SAMPLES])
    dev = d.device
    out = {"t_starts": torch.empty(total + offset, dtype=torch.float64, device=dev)[offset:],
           "t_ends": torch.empty(total + offset, dtype=torch.float64, device=dev)[offset:],
           "ray_indices": torch.empty(total + offset, dtype=torch.int32, device=dev)[offset:],
           "cells": torch.empty(total + offset, dtype=torch.int32, device=dev)[offset:],
           "levels": torch.empty(total + offset, dtype=torch.uint8, device=dev)[offset:]}
    s.write(d, packed, total, out=out)
    torch.cuda.synchronize()
    return packed.cpu().numpy(), {k: v.cpu().numpy() for k, v in out.items()}


def _check(got, want, what):
    pi, o = got
    assert np.array_equal(pi, want.packed_info), what
    assert np.array_equal(bits64(o["t_starts"]), bits64(want.t_starts)), what
    assert np.array_equal(bits64(o["t_ends"]), bits64(want.t_ends)), what
    assert np.array_equal(o["ray_indices"], want.ray_indices), what
    assert np.array_equal(o["cells"].view(np.uint32), want.cells), what
    assert np.array_equal(o["levels"], want.levels), what


@pytest.mark.parametrize("offset", [0, 1])
@pytest.mark.parametrize("slab", [None, "1"])
def test_output_parallel_batches(P, oracle, monkeypatch, offset, slab):
    if slab is not None:
        monkeypatch.setenv("SOGK_SLAB", slab)
    t, g = _tile_grid(P)
    rays = _rays(P, t, 4000, seed=17)
    for dt in (1.0 / 128.0, 1.0 / 448.0, 0.013):
        sched = P.StepSchedule.constant(dt)
        for kernel in (SKIP, BRANCH):
            want = oracle_sample(oracle, [g], HDDA, kernel, sched, rays)
            assert want.total > 0
            runs = np.diff(np.flatnonzero(np.diff(want.cells.astype(np.int64), prepend=-1)))
            assert runs.size and runs.max() > 8, "the grid must produce long runs"
            got = _run(P, g, t, kernel, sched, rays, offset)
            _check(got, want, f"dt={dt} kernel={kernel} offset={offset} slab={slab}")
