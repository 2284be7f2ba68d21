"""GPU VDB build (K1) parity: byte-identical SOG1 export vs the oracle's
serialize_sparse(build_sparse(dense)) (io.hpp:161-181, sparse.hpp:333-371), exhaustive
occupancy round trip, memory accounting, SOG0/SOG1 load and the io_error paths."""
import numpy as np
import pytest

from parity_util import host_grid, scene_grid

pytestmark = pytest.mark.gpu


def _vdb(P, g):
    return P.build_sparse(P.DenseGrid(P.GridTransform(g.res, g.wmin, g.voxel), g.bits))


def _cases(P):
    out = []
    for kind in ("shell", "blobs", "sponge", "random"):
        out.append((kind, scene_grid(P, kind, 128, seed=1, fraction=0.02)))
    for res, seed, bf, nf in [((32, 32, 32), 1, 0.3, 0.02), ((11, 5, 9), 9, 0.4, 0.0),
                              ((144, 144, 144), 77, 0.02, 0.001), ((24, 24, 24), 3, 0.0, 0.0),
                              ((8, 16, 24), 4, 0.5, 0.01), ((130, 7, 257), 6, 0.05, 0.001)]:
        t = P.GridTransform(res, (-1.0, -1.0, -1.0), 2.0 / res[0])
        out.append((f"blocky{res}", host_grid(P, t, P.random_blocky_grid(t, seed, bf, nf))))
    t = P.GridTransform.cube(128, (-1, -1, -1), 2.0)
    out.append(("empty", host_grid(P, t, np.zeros(t.payload_bytes(), np.uint8))))
    out.append(("full", host_grid(P, t, np.full(t.payload_bytes(), 0xFF, np.uint8))))
    t32 = P.GridTransform.cube(32, (-1, -1, -1), 2.0)  # padded: a full 32^3 is NOT a root tile
    out.append(("full32", host_grid(P, t32, np.full(t32.payload_bytes(), 0xFF, np.uint8))))
    return out


def test_sog1_bytes_match_oracle(P, oracle):
    for name, g in _cases(P):
        v = _vdb(P, g)
        got = P.serialize_sparse(v)
        want = oracle.sog1(g)
        assert got == want, name
        assert P.memory_bytes(v) == len(want), name
        assert v.leaf_count() == oracle.L.og_sparse_leaf_count(oracle.sparse(g)), name


def test_to_dense_round_trip_and_idempotence(P):
    for name, g in _cases(P):
        v = _vdb(P, g)
        assert np.array_equal(v.payload(), g.bits), name
        again = P.build_sparse(P.DenseGrid(v.transform(), v.payload()))
        assert P.serialize_sparse(again) == P.serialize_sparse(v), name


def test_512_blobs(P, oracle):
    g = scene_grid(P, "blobs", 512, seed=1)
    v = _vdb(P, g)
    assert P.serialize_sparse(v) == oracle.sog1(g)
    assert v.root_size() == 64


def test_sog_loaders(P, oracle):
    g = scene_grid(P, "sponge", 64, seed=1)
    want = oracle.sog1(g)
    v = P.deserialize_sparse(want)
    assert P.serialize_sparse(v) == want
    assert np.array_equal(v.payload(), g.bits)
    d = P.DenseGrid(P.GridTransform(g.res, g.wmin, g.voxel), g.bits)
    s0 = P.serialize_dense(d)
    assert P.serialize_dense(P.deserialize_dense(s0)) == s0
    for bad, code in [(b"XXXX" + want[4:], "bad magic"), (want[:4] + b"\x02\0\0\0" + want[8:], "bad version"),
                      (want[:-5], "truncated"), (want + b"\0", "corrupt")]:
        with pytest.raises(P.IoError) as e:
            P.deserialize_sparse(bad)
        assert e.value.code == code
    with pytest.raises(P.IoError):
        P.deserialize_dense(s0[:-1])
