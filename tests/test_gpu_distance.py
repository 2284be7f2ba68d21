"""GPU build_distance (exact separable chessboard transform) vs the oracle's chamfer
(bit-exact int32), incl. odd resolutions, an empty grid and 512^3."""
import numpy as np
import pytest

from parity_util import host_grid

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("res,seed,kind", [((32, 32, 32), 1, "blobs"), ((128, 128, 128), 1, "shell"),
                                           ((128, 128, 128), 1, "random"), ((11, 5, 9), 9, None),
                                           ((40, 24, 16), 5, None), ((144, 144, 144), 77, None)])
def test_distance_field(P, oracle, res, seed, kind):
    t = P.GridTransform(res, (-1.0, -1.0, -1.0), 2.0 / res[0])
    bits = P.generate_scene(kind, t, seed=seed, fraction=0.02)[0] if kind else \
        P.random_blocky_grid(t, seed, 0.02, 0.001)
    g = host_grid(P, t, bits)
    d = P.build_distance(P.DenseGrid(t, bits))
    want, ae = oracle.distance_field(g)
    assert np.array_equal(d.distances(), want)
    assert d.all_empty() == ae
    assert d.memory_bytes() == 4 * t.voxel_count()


def test_distance_empty(P, oracle):
    t = P.GridTransform((7, 9, 5), (0.0, 0.0, 0.0), 1.0)
    bits = np.zeros(t.payload_bytes(), np.uint8)
    d = P.build_distance(P.DenseGrid(t, bits))
    want, ae = oracle.distance_field(host_grid(P, t, bits))
    assert ae and d.all_empty() and np.array_equal(d.distances(), want)


def test_distance_512(P):
    """512^3 blobs (cfg4's grid): exact L-inf distance checked on sampled voxels by brute force."""
    t = P.GridTransform.cube(512, (-1.0, -1.0, -1.0), 2.0)
    bits, _ = P.generate_scene("blobs", t, seed=1)
    d = P.build_distance(P.DenseGrid(t, bits)).distances()
    occ = np.unpackbits(bits, bitorder="little")[: 512 ** 3].reshape(512, 512, 512).astype(bool)
    pts = np.argwhere(occ)  # (z, y, x)
    rng = np.random.default_rng(3)
    for z, y, x in rng.integers(0, 512, size=(40, 3)):
        ref = int(np.abs(pts - np.array([z, y, x])).max(axis=1).min())
        assert d[z, y, x] == ref


@pytest.mark.parametrize("res", [(1500, 3, 4), (4, 1500, 3), (3, 4, 1500), (2047, 2, 2)])
def test_distance_long_lines(P, oracle, res):
    """Lines up to the 2047-voxel limit on each axis (shared-memory sizing of every pass)."""
    t = P.GridTransform(res, (0.0, 0.0, 0.0), 1.0)
    bits = P.random_grid(t, 11, 0.003)
    d = P.build_distance(P.DenseGrid(t, bits))
    want, ae = oracle.distance_field(host_grid(P, t, bits))
    assert np.array_equal(d.distances(), want) and d.all_empty() == ae


def test_builds_on_side_stream_then_read(P):
    """Grid builds are stream-ordered (pool storage, no sync): host reads right after a build
    on another stream wait for it (build-completion event), and rebuilt grids reusing pool
    blocks give identical results."""
    import torch

    t = P.GridTransform.cube(128, (-1.0, -1.0, -1.0), 2.0)
    bits, _ = P.generate_scene("shell", t, seed=1)
    dense = P.DenseGrid(t, bits)
    want_d = P.build_distance(dense).distances()
    want_s = P.serialize_sparse(P.build_sparse(dense))
    side = torch.cuda.Stream()
    for _ in range(5):
        with torch.cuda.stream(side):
            g = P.build_distance(dense, stream=side)
            v = P.build_sparse(dense, stream=side)
        assert np.array_equal(g.distances(), want_d)
        assert P.serialize_sparse(v) == want_s
        del g, v
    P.release_workspaces()  # trims the pool
    assert np.array_equal(P.build_distance(dense).distances(), want_d)
