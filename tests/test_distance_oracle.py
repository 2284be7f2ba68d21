"""The CD analyzer's checkers (CPU only): build_distance and CdTraversal sampling of the oracle
pinned to the unmodified reference (distance.hpp:45-103, traversal.hpp:270-337,
sampling.hpp:198-212), on scene grids, blocky grids, odd resolutions and an empty grid."""
import numpy as np
import pytest

from oracle_bindings import BRANCH, CD, CONSTANT, LINEAR, SKIP, Grid


def _grid(P, res, seed, kind=None, bf=0.1, nf=0.01):
    t = P.GridTransform(res, (-1.0, -1.0, -1.0), 2.0 / res[0])
    bits = P.generate_scene(kind, t, seed=seed)[0] if kind else P.random_blocky_grid(t, seed, bf, nf)
    return Grid(tuple(t.resolution), tuple(t.world_min), t.voxel_size, np.asarray(bits, np.uint8))


CASES = [((32, 32, 32), 1, "blobs"), ((24, 24, 24), 2, "shell"), ((16, 16, 16), 5, "random"),
         ((11, 5, 9), 9, None), ((40, 24, 16), 5, None)]


@pytest.mark.parametrize("res,seed,kind", CASES)
def test_distance_field_matches_reference(P, oracle, reflib, res, seed, kind):
    g = _grid(P, res, seed, kind)
    a, ea = oracle.distance_field(g)
    b, eb = reflib.distance_field(g)
    assert np.array_equal(a, b) and ea == eb


def test_distance_all_empty(P, oracle, reflib):
    g = Grid((7, 9, 5), (0.0, 0.0, 0.0), 1.0, np.zeros((7 * 9 * 5 + 7) // 8, np.uint8))
    a, ea = oracle.distance_field(g)
    b, eb = reflib.distance_field(g)
    assert ea and eb and np.array_equal(a, b) and int(a.max()) == 9  # sentinel max(resolution)


@pytest.mark.parametrize("res,seed,kind", CASES)
def test_cd_sampler_matches_reference(P, oracle, reflib, res, seed, kind):
    g = _grid(P, res, seed, kind)
    t = P.GridTransform(g.res, g.wmin, g.voxel)
    rays = P.random_rays(t, 400, seed=seed + 3)
    for sk, dt0, gr in ((CONSTANT, 0.5 * g.voxel, 0.0), (LINEAR, 0.011, 1.0 / 128.0)):
        for k in (BRANCH, SKIP):
            got = oracle.sample(oracle.sampler([g], CD, k, sk, dt0, gr), rays)
            want = reflib.sampler([g], CD, k, sk, dt0, gr).sample(rays)
            assert np.array_equal(got.packed_info, want.packed_info)
            assert np.array_equal(got.t_starts.view(np.uint64), want.t_starts.view(np.uint64))
            assert np.array_equal(got.t_ends.view(np.uint64), want.t_ends.view(np.uint64))
            assert np.array_equal(got.cells, want.cells) and np.array_equal(got.levels, want.levels)
            assert np.array_equal(got.counters, want.counters)


def test_cd_cascade_matches_reference(P, oracle, reflib):
    base = P.GridTransform.cube(32, (-1.0, -1.0, -1.0), 2.0)
    lv = [Grid(tuple(t.resolution), tuple(t.world_min), t.voxel_size, np.asarray(b, np.uint8))
          for t, b in P.build_dense_cascade("blobs", base, 4, seed=1)]
    rays = P.random_rays(P.GridTransform(lv[-1].res, lv[-1].wmin, lv[-1].voxel), 500, 3)
    for k in (BRANCH, SKIP):
        got = oracle.sample(oracle.sampler(lv, CD, k, LINEAR, 2.0 / 64, 1.0 / 256), rays)
        want = reflib.sampler(lv, CD, k, LINEAR, 2.0 / 64, 1.0 / 256).sample(rays)
        assert np.array_equal(got.packed_info, want.packed_info)
        assert np.array_equal(got.t_starts.view(np.uint64), want.t_starts.view(np.uint64))
        assert np.array_equal(got.cells, want.cells) and np.array_equal(got.levels, want.levels)
        assert np.array_equal(got.counters, want.counters)


def test_cd_events_match_reference(P, oracle, reflib):
    g = _grid(P, (32, 32, 32), 1, "blobs")
    t = P.GridTransform(g.res, g.wmin, g.voxel)
    s = oracle.sampler([g], CD, SKIP, CONSTANT, 0.5 * g.voxel)
    rs = reflib.sampler([g], CD, SKIP, CONSTANT, 0.5 * g.voxel)
    for r in P.random_rays(t, 100, seed=21):
        na, ea, ca = oracle.events(s, r)
        nb, eb, cb = rs.events(r)
        assert na == nb and ea == eb and np.array_equal(ca, cb)
