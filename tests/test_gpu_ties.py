"""Tie / near-tie stress of the node analyzers (HDDA, CD) and the branch kernel's probe: rays
through voxel corners, edges and faces with axis-aligned and diagonal directions on fully mixed
grids (every crossing an exact or near tie, the reference's degenerate re-derivation and its
edge-crossing spin), plus iid random grids at the occupancies of the cfg5 sweep; every output
(events, samples, cells, counters, spin flags) is compared bit for bit with the C oracle.
(This suite found the branch kernel's probe on out-of-grid root-tile events, step_event.)"""
import itertools
import math

import numpy as np
import pytest
import torch

from oracle_bindings import BRANCH, CD, HDDA, SKIP
from parity_util import assert_packed_equal, gpu_sample, host_grid, oracle_sample

pytestmark = pytest.mark.gpu


def _tie_rays(res, n_per_dir=400, seed=3):
    """Rays from dyadic points on voxel corners / edges / faces, directions with exact ties."""
    rng = np.random.default_rng(seed)
    dirs = []
    for v in [(1, 0, 0), (1, 1, 0), (1, 1, 1), (1, 2, 2), (3, 4, 0), (2, 1, 0), (1, 1, 2), (4, 4, 7)]:
        for p in set(itertools.permutations(v)):
            for sg in itertools.product((1, -1), repeat=3):
                d = np.array([p[i] * sg[i] for i in range(3)], np.float64)
                dirs.append(d / math.sqrt(float(d @ d)))
    dirs = np.unique(np.round(np.array(dirs), 15), axis=0)
    rays = []
    for d in dirs:
        # start outside the box on the back side of the direction, on lattice points (corners),
        # edge midpoints and face centres of the voxel grid
        base = rng.integers(0, res + 1, size=(n_per_dir, 3)).astype(np.float64)
        frac = rng.choice([0.0, 0.5, 0.25], size=(n_per_dir, 3))
        o = base + frac - d * (res * 2.0)
        for q in o:
            rays.append([*q, *d, 0.0, 1e6])
    return np.array(rays, np.float64)


@pytest.mark.parametrize("fill", ["checker", "iid30", "iid2"])
def test_tie_rays_on_mixed_grids(P, oracle, fill):
    res = 32
    t = P.GridTransform((res, res, res), (0.0, 0.0, 0.0), 1.0)  # unit voxels: lattice = planes
    if fill == "checker":
        bits = np.zeros(t.payload_bytes(), np.uint8)
        for z in range(res):
            for y in range(res):
                for x in range(res):
                    if (x + y + z) % 2 == 0:
                        i = (z * res + y) * res + x
                        bits[i >> 3] |= 1 << (i & 7)
    else:
        bits = P.random_grid(t, 7, 0.30 if fill == "iid30" else 0.02)
    g = host_grid(P, t, bits)
    rays = _tie_rays(res)
    for an in (HDDA, CD):
        for k in (SKIP, BRANCH):
            for sched in (P.StepSchedule.constant(0.25), P.StepSchedule.constant(0.3)):
                got = gpu_sample(P, [g], an, k, sched, rays, spin_cap=64)
                want = oracle_sample(oracle, [g], an, k, sched, rays)
                assert_packed_equal(got, want, f"{fill} an={an} k={k} dt={sched.dt0}")


@pytest.mark.parametrize("frac", [0.005, 0.05, 0.2, 0.5])
def test_iid_random_cfg5_shapes(P, oracle, frac):
    t = P.GridTransform.cube(128, (-1.0, -1.0, -1.0), 2.0)
    bits = P.random_grid(t, 11, frac)
    g = host_grid(P, t, bits)
    rays = np.concatenate([P.make_probe_rays(t, 60000, 5), P.random_rays(t, 20000, 6)])
    sched = P.StepSchedule.constant(0.5 * t.voxel_size)
    for an in (HDDA, CD):
        got = gpu_sample(P, [g], an, SKIP, sched, rays)
        want = oracle_sample(oracle, [g], an, SKIP, sched, rays)
        assert_packed_equal(got, want, f"iid {frac} an={an}")
