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
