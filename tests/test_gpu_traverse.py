"""The traverse entry points on the GPU (sogk_traverse_count / _write / _host, sogk_grid_query):
event streams of DdaTraversal / HddaTraversal / CdTraversal / CascadeTraversal (collect_events,
traversal.hpp:120-359, sampling.hpp:305-415) and SparseGrid::query (sparse.hpp:163-171),
bit for bit against the reference's golden vectors, the unmodified reference (oracle/_ref)
and the C oracle, plus the reference unit suite's known answers re-expressed
(test_traversal.cpp:35-70,135-185,327-340; test_vdb_tree.cpp query cases)."""
import numpy as np
import pytest
import torch

from oracle_bindings import CD, DDA, HDDA, SKIP, Grid
from parity_util import bits64, gpu_grids, host_grid, scene_grid

pytestmark = pytest.mark.gpu


def _gpu_events(P, levels, an, rays, cascade=False):
    s = P.Sampler(gpu_grids(P, levels, an), an, SKIP, P.StepSchedule.constant(1.0), cascade=cascade)
    t = s.traverse(torch.from_numpy(np.ascontiguousarray(rays).reshape(-1, 8)).cuda())
    torch.cuda.synchronize()
    info = t.event_info.cpu().numpy()
    return info, t.host_events(), t.status.cpu().numpy(), t.counters.cpu().numpy(), t.stats


def _rows(ev):
    return (np.stack([ev["ijk"][:, 0], ev["ijk"][:, 1], ev["ijk"][:, 2], ev["level"], ev["occupied"],
                      ev["grid_level"]], 1).astype(np.int32),
            np.stack([ev["t0"], ev["t1"]], 1))


def test_events_match_reference_golden(P):
    gold = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                              "reference_golden.npz"))
    g = Grid(tuple(gold["scene0_res"]), tuple(gold["scene0_wmin"]), float(gold["scene0_voxel"]),
             gold["scene0_bits"])
    rays = gold["rays_random"][:20]
    for an in (DDA, HDDA):
        info, ev, st, ctr, _ = _gpu_events(P, [g], an, rays)
        n = gold[f"events_an{an}_n"]
        assert np.array_equal(info[:, 1], n[:, 0])
        assert np.array_equal(ctr[:, 0], n[:, 1]) and np.array_equal(ctr[:, 1], n[:, 2])
        iv, tv = _rows(ev)
        assert np.array_equal(iv, gold[f"events_an{an}_ev"])
        assert np.array_equal(bits64(tv), bits64(gold[f"events_an{an}_t"]))


def _cmp_ref(P, reflib, levels, an, rays, cascade=False, what=""):
    info, ev, st, ctr, _ = _gpu_events(P, levels, an, rays, cascade)
    rs = reflib.sampler(levels, an, SKIP, 0, 1.0, 0.0, cascade=cascade)
    for i, r in enumerate(rays):
        if st[i] == 2:  # the reference never returns on this ray (checked against the oracle below)
            continue
        n, evs, c = rs.events(r)
        o, k = info[i]
        assert k == n, f"{what} ray {i}: {k} events, reference {n}"
        got = ev[o:o + k]
        for j, e in enumerate(evs):
            g = got[j]
            assert (tuple(int(x) for x in g["ijk"]), int(g["level"]), int(g["occupied"]), int(g["grid_level"])) == \
                   (e[0], e[1], e[4], e[5]), f"{what} ray {i} event {j}"
            assert np.float64(g["t0"]).view(np.uint64) == np.float64(e[2]).view(np.uint64)
            assert np.float64(g["t1"]).view(np.uint64) == np.float64(e[3]).view(np.uint64)
        assert (ctr[i, 0], ctr[i, 1]) == (c[0], c[1]), f"{what} ray {i} counters"


@pytest.mark.parametrize("kind", ["shell", "blobs", "random"])
def test_events_vs_reference_128(P, reflib, kind):
    g = scene_grid(P, kind, 128, seed=2, fraction=0.03)
    t = P.GridTransform(g.res, g.wmin, g.voxel)
    rays = np.concatenate([P.random_rays(t, 250, seed=9),
                           P.Camera((1.9, 1.4, 2.3), (0, 0, 0), (0, 1, 0), 42.0, 40, 30).rays()])
    for an in (DDA, HDDA, CD):
        _cmp_ref(P, reflib, [g], an, rays, what=f"{kind} an={an}")


def test_cascade_events_vs_reference(P, reflib):
    lv = [host_grid(P, tt, b) for tt, b in
          P.build_dense_cascade("blobs", P.GridTransform.cube(64, (-1, -1, -1), 2.0), 4, seed=1)]
    rays = P.Camera((1.9, 1.4, 2.3), (0, 0, 0), (0, 1, 0), 42.0, 30, 24).rays()
    rays = np.concatenate([rays, P.random_rays(P.GridTransform(lv[-1].res, lv[-1].wmin, lv[-1].voxel), 200, 3)])
    for an in (DDA, HDDA, CD):
        _cmp_ref(P, reflib, lv, an, rays, cascade=True, what=f"cascade an={an}")


def test_events_vs_oracle_batch_and_spin(P, oracle):
    """A larger batch against the C restatement (events, counters, status), including the
    1297x840 u == 0 column where HddaTraversal never returns (status UNDEFINED, no events)."""
    g = scene_grid(P, "shell", 128, seed=1)
    cam = P.Camera((1.9, 1.4, 2.3), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, 1297, 840)
    allr = cam.rays()
    rays = allr[np.array([py * 1297 + px for py in range(0, 840, 2) for px in (647, 648, 649)])]
    for an in (DDA, HDDA, CD):
        info, ev, st, ctr, stats = _gpu_events(P, [g], an, rays)
        s = oracle.sampler([g], an, SKIP, 0, 1.0)
        und = 0
        for i, r in enumerate(rays):
            n, evs, c = oracle.events(s, r)
            if n == -1:  # the oracle's capped detector: the reference spins on this ray
                assert st[i] == 2 and info[i, 1] == 0
                und += 1
                continue
            assert st[i] == 0 and info[i, 1] == n
            o = info[i, 0]
            for j, e in enumerate(evs):
                gg = ev[o + j]
                assert tuple(int(x) for x in gg["ijk"]) == e[0] and int(gg["level"]) == e[1]
                assert gg["t0"] == e[2] and gg["t1"] == e[3] and int(gg["occupied"]) == e[4]
            assert (ctr[i, 0], ctr[i, 1]) == (c[0], c[1])
        assert int(stats[2]) == und
        if an == HDDA:
            assert und > 0


def test_known_answers_and_dump_trace(P):
    # test_traversal.cpp:35-51 -- dda walks an axis ray voxel by voxel
    t4 = P.GridTransform((4, 4, 4), (0.0, 0.0, 0.0), 1.0)
    bits = np.zeros(8, np.uint8)
    bits[0] |= 1 << 2  # voxel (2, 0, 0)
    d = P.DenseGrid(t4, bits)
    ray = [-1.0, 0.5, 0.5, 1.0, 0.0, 0.0, 0.0, 100.0]
    ev, lk, sp = P.collect_events(d, ray)
    assert len(ev) == 4 and lk == 4 and sp == 4
    assert [tuple(e["ijk"]) for e in ev] == [(i, 0, 0) for i in range(4)]
    assert list(ev["t0"]) == [1.0, 2.0, 3.0, 4.0] and list(ev["t1"]) == [2.0, 3.0, 4.0, 5.0]
    assert list(ev["occupied"]) == [0, 0, 1, 0]
    # :53-70 -- exact corner ties collapse, no zero-length events
    r2 = 1.0 / np.sqrt(2.0)
    ev, _, _ = P.collect_events(P.DenseGrid(t4, np.zeros(8, np.uint8)), [-0.5, -0.5, 0.5, r2, r2, 0.0, 0.0, 100.0])
    assert [tuple(e["ijk"]) for e in ev] == [(i, i, 0) for i in range(4)]
    assert np.allclose(ev["t1"] - ev["t0"], np.sqrt(2.0))
    # :327-340 -- the trace dump format
    b1 = np.zeros(8, np.uint8)
    b1[0] |= 1 << 1
    ev, _, _ = P.collect_events(P.DenseGrid(t4, b1), ray)
    assert P.dump_trace(ev) == ("leaf_voxel\t0,0,0\t1\t2\t0\n" "leaf_voxel\t1,0,0\t2\t3\t1\n"
                                "leaf_voxel\t2,0,0\t3\t4\t0\n" "leaf_voxel\t3,0,0\t4\t5\t0\n")
    # :135-160 -- hdda merges an occupied leaf tile into one event
    t = P.GridTransform.cube(128, (0.0, 0.0, 0.0), 128.0)
    bits = np.zeros(t.payload_bytes(), np.uint8)
    for z in range(8):
        for y in range(8):
            for x in range(8):
                i = (z * 128 + y) * 128 + x
                bits[i >> 3] |= 1 << (i & 7)
    sp = P.build_sparse(P.DenseGrid(t, bits))
    ev, _, _ = P.collect_events(sp, [-1.0, 4.5, 4.5, 1.0, 0.0, 0.0, 0.0, 1000.0])
    occ = ev[ev["occupied"] == 1]
    assert len(occ) == 1 and int(occ[0]["level"]) == 1 and tuple(occ[0]["ijk"]) == (0, 0, 0)
    assert occ[0]["t1"] - occ[0]["t0"] == 8.0
    assert all(int(e["level"]) >= 1 for e in ev[ev["occupied"] == 0])
    # :162-185 -- checkerboard 16^3: hdda events == dda events bit for bit (random_ray, seed 77)
    t16 = P.GridTransform.cube(16, (-1.0, -1.0, -1.0), 2.0)
    cb = np.zeros(t16.payload_bytes(), np.uint8)
    for z in range(16):
        for y in range(16):
            for x in range(16):
                if (x + y + z) % 2 == 0:
                    i = (z * 16 + y) * 16 + x
                    cb[i >> 3] |= 1 << (i & 7)
    dn = P.DenseGrid(t16, cb)
    spc = P.build_sparse(dn)
    assert spc.leaf_count() == 8
    rays = P.random_rays(t16, 50, 77)
    sd = P.Sampler([dn], DDA, SKIP, P.StepSchedule.constant(1.0)).traverse_host(rays)
    sh = P.Sampler([spc], HDDA, SKIP, P.StepSchedule.constant(1.0)).traverse_host(rays)
    assert np.array_equal(sd.event_info, sh.event_info)
    for f in ("ijk", "occupied"):
        assert np.array_equal(sd.events[f], sh.events[f])
    assert np.array_equal(bits64(sd.events["t0"]), bits64(sh.events["t0"]))
    assert np.array_equal(bits64(sd.events["t1"]), bits64(sh.events["t1"]))


def test_query_vs_oracle_and_known_answers(P, oracle):
    import ctypes as C

    for kind, res in (("shell", 128), ("blobs", 144), ("random", 64)):
        t = P.GridTransform.cube(res, (-1.0, -1.0, -1.0), 2.0)
        bits, _ = P.generate_scene(kind, t, seed=3, fraction=0.05)
        g = host_grid(P, t, bits)
        vdb = P.build_sparse(P.DenseGrid(t, bits))
        rng = np.random.default_rng(5)
        pts = rng.integers(-300, res + 300, size=(20000, 3)).astype(np.int32)
        pts[:5000] = rng.integers(0, res, size=(5000, 3))
        got = P.query(vdb, pts)
        h = oracle.sparse(g)
        for i in range(0, pts.shape[0], 7):
            lvl, ext = C.c_int32(0), C.c_int32(0)
            org = np.zeros(3, np.int32)
            occ = oracle.L.og_sparse_query(h, pts[i], C.byref(lvl), org, C.byref(ext))
            q = got[i]
            assert (int(q["occupied"]), int(q["level"]), tuple(int(x) for x in q["origin"]), int(q["extent"])) == \
                   (occ, lvl.value, tuple(int(x) for x in org), ext.value), (kind, pts[i])
        dq = P.query(P.DenseGrid(t, bits), pts[:5000])
        for i in range(0, 5000, 13):
            assert int(dq[i]["occupied"]) == oracle.L.og_dense_voxel_at(oracle.dense(g), pts[i])
    # test_vdb_tree.cpp: out of bounds (-3, 5, 5) -> root_tile at (-128, 0, 0), extent 128
    t = P.GridTransform.cube(32, (0.0, 0.0, 0.0), 32.0)
    q = P.query(P.build_sparse(P.DenseGrid(t, np.full(t.payload_bytes(), 0xFF, np.uint8))), [[-3, 5, 5]])[0]
    assert (int(q["occupied"]), int(q["level"]), tuple(q["origin"]), int(q["extent"])) == (0, 3, (-128, 0, 0), 128)
