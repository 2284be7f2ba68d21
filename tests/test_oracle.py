"""The CPU oracle (oracle/sog_oracle.c) pinned to the reference.

(1) golden vectors produced by the unmodified reference headers
    (tests/golden/make_golden.py -> reference_golden.npz);
(2) known-answer tests of the reference's own unit suite, re-expressed
    (proj/tests/unit/test_traversal.cpp, test_sampling.cpp, test_vdb_tree.cpp);
(3) randomized cross-checks against oracle/_ref when it is built here.
"""
import math
import os

import numpy as np
import pytest

from oracle_bindings import BRANCH, CONSTANT, DDA, HDDA, LINEAR, SKIP, Grid

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def _grid(gold, prefix) -> Grid:
    return Grid(tuple(int(x) for x in gold[f"{prefix}_res"]), tuple(gold[f"{prefix}_wmin"]),
                float(gold[f"{prefix}_voxel"]), gold[f"{prefix}_bits"])


def _eq64(a, b):
    return np.array_equal(np.asarray(a, np.float64).view(np.uint64), np.asarray(b, np.float64).view(np.uint64))


def test_sampler_cases_match_reference(oracle, gold):
    rays_by = {0: gold["rays_random"], 1: gold["rays_camera"]}
    for ci in range(int(gold["n_cases"])):
        si, rk, an, k, sk, dt, gr = gold[f"case{ci}_args"]
        g = _grid(gold, f"scene{int(si)}")
        s = oracle.sampler([g], int(an), int(k), int(sk), dt, gr)
        p = oracle.sample(s, rays_by[int(rk)])
        assert np.array_equal(p.packed_info, gold[f"case{ci}_packed_info"]), ci
        assert _eq64(p.t_starts, gold[f"case{ci}_t_starts"]), ci
        assert _eq64(p.t_ends, gold[f"case{ci}_t_ends"]), ci
        assert np.array_equal(p.cells, gold[f"case{ci}_cells"]), ci
        assert np.array_equal(p.levels, gold[f"case{ci}_levels"]), ci
        assert np.array_equal(p.counters, gold[f"case{ci}_counters"]), ci


def test_cascade_cases_match_reference(oracle, gold):
    lv = [_grid(gold, f"casc{b}") for b in range(4)]
    for an, k in ((DDA, BRANCH), (HDDA, SKIP)):
        p = oracle.sample(oracle.sampler(lv, an, k, LINEAR, 0.013, 1.0 / 256), gold["casc_rays"])
        pre = f"casc_an{an}k{k}"
        assert np.array_equal(p.packed_info, gold[f"{pre}_packed_info"])
        assert _eq64(p.t_starts, gold[f"{pre}_t_starts"])
        assert np.array_equal(p.cells, gold[f"{pre}_cells"])
        assert np.array_equal(p.levels, gold[f"{pre}_levels"])
        assert np.array_equal(p.counters, gold[f"{pre}_counters"])


def test_event_streams_match_reference(oracle, gold):
    g = _grid(gold, "scene0")
    for an in (DDA, HDDA):
        s = oracle.sampler([g], an, SKIP, CONSTANT, 0.03)
        evs, ts = [], []
        ns = []
        for r in gold["rays_random"][:20]:
            n, ev, ctr = oracle.events(s, r)
            ns.append((n, ctr[0], ctr[1]))
            for e in ev:
                evs.append([*e[0], e[1], e[4], e[5]])
                ts.append([e[2], e[3]])
        assert np.array_equal(np.asarray(ns), gold[f"events_an{an}_n"])
        assert np.array_equal(np.asarray(evs, np.int32), gold[f"events_an{an}_ev"])
        assert _eq64(np.asarray(ts), gold[f"events_an{an}_t"])


def test_sog1_matches_reference(oracle, gold):
    for pre in ["scene0", "scene1", "scene2", "scene3", "scene4", "blocky0", "blocky1"]:
        assert oracle.sog1(_grid(gold, pre)) == gold[f"{pre}_sog1"].tobytes(), pre


# ---------------------------------------------------------------------------
# reference unit-suite known answers
# ---------------------------------------------------------------------------
def _unit4(bits_set=()):
    bits = np.zeros(8, np.uint8)
    for (x, y, z) in bits_set:
        i = (z * 4 + y) * 4 + x
        bits[i >> 3] |= 1 << (i & 7)
    return Grid((4, 4, 4), (0.0, 0.0, 0.0), 1.0, bits)


def test_dda_axis_ray(oracle):
    """test_traversal.cpp:35-51"""
    s = oracle.sampler([_unit4([(2, 0, 0)])], DDA, SKIP, CONSTANT, 0.5)
    n, ev, ctr = oracle.events(s, [-1.0, 0.5, 0.5, 1.0, 0.0, 0.0, 0.0, 100.0])
    assert n == 4 and list(ctr) == [4, 4]
    for i, e in enumerate(ev):
        assert e[0] == (i, 0, 0) and e[1] == 0
        assert math.isclose(e[2], 1.0 + i) and math.isclose(e[3], 2.0 + i)
        assert e[4] == (1 if i == 2 else 0)


def test_dda_diagonal_corner_ties(oracle):
    """test_traversal.cpp:53-70: exact corner ties collapse, no zero-length events"""
    s = oracle.sampler([_unit4()], DDA, SKIP, CONSTANT, 0.5)
    r = 1.0 / math.sqrt(2.0)
    n, ev, _ = oracle.events(s, [-0.5, -0.5, 0.5, r, r, 0.0, 0.0, 100.0])
    assert n == 4
    for i, e in enumerate(ev):
        assert e[0] == (i, i, 0)
        assert math.isclose(e[3] - e[2], math.sqrt(2.0), rel_tol=1e-12)


def test_no_clip_no_events(oracle):
    """test_traversal.cpp:96-103"""
    s = oracle.sampler([_unit4()], DDA, SKIP, CONSTANT, 0.5)
    n, ev, ctr = oracle.events(s, [10.0, 10.0, 10.0, 1.0, 0.0, 0.0, 0.0, 100.0])
    assert n == 0 and ctr[1] == 0


def test_trace_dump_format(oracle):
    """test_traversal.cpp:327-340 golden dump_trace text"""
    s = oracle.sampler([_unit4([(1, 0, 0)])], DDA, SKIP, CONSTANT, 0.5)
    _, ev, _ = oracle.events(s, [-1.0, 0.5, 0.5, 1.0, 0.0, 0.0, 0.0, 100.0])
    names = ["leaf_voxel", "leaf_tile", "internal_tile", "root_tile"]
    text = "".join(f"{names[e[1]]}\t{e[0][0]},{e[0][1]},{e[0][2]}\t{e[2]:.17g}\t{e[3]:.17g}\t{e[4]}\n" for e in ev)
    assert text == ("leaf_voxel\t0,0,0\t1\t2\t0\n"
                    "leaf_voxel\t1,0,0\t2\t3\t1\n"
                    "leaf_voxel\t2,0,0\t3\t4\t0\n"
                    "leaf_voxel\t3,0,0\t4\t5\t0\n")


def _unit128_block(x0s, y0=0, z0=0):
    bits = np.zeros(128 ** 3 // 8, np.uint8)
    for x0 in x0s:
        for z in range(8):
            for y in range(8):
                for x in range(8):
                    i = ((z + z0) * 128 + (y + y0)) * 128 + x0 + x
                    bits[i >> 3] |= 1 << (i & 7)
    return Grid((128, 128, 128), (0.0, 0.0, 0.0), 1.0, bits)


def test_hdda_merges_leaf_tile(oracle):
    """test_traversal.cpp:135-160: one occupied 8-block -> a single leaf_tile event of length 8"""
    s = oracle.sampler([_unit128_block([0])], HDDA, SKIP, CONSTANT, 0.5)
    _, ev, _ = oracle.events(s, [-1.0, 4.5, 4.5, 1.0, 0.0, 0.0, 0.0, 1000.0])
    occ = [e for e in ev if e[4]]
    assert len(occ) == 1 and occ[0][1] == 1 and occ[0][0] == (0, 0, 0)
    assert math.isclose(occ[0][3] - occ[0][2], 8.0)
    assert all(e[1] >= 1 for e in ev if not e[4])


def test_hdda_equals_dda_on_checkerboard(oracle, P):
    """test_traversal.cpp:162-185: every leaf mixed -> HDDA events == DDA events bit-exactly"""
    bits = np.zeros(16 ** 3 // 8, np.uint8)
    for z in range(16):
        for y in range(16):
            for x in range(16):
                if (x + y + z) % 2 == 0:
                    i = (z * 16 + y) * 16 + x
                    bits[i >> 3] |= 1 << (i & 7)
    g = Grid((16, 16, 16), (-1.0, -1.0, -1.0), 2.0 / 16, bits)
    assert oracle.L.og_sparse_leaf_count(oracle.sparse(g)) == 8
    rays = P.random_rays(P.GridTransform.cube(16, (-1, -1, -1), 2.0), 50, 77)
    sd = oracle.sampler([g], DDA, SKIP, CONSTANT, 0.1)
    sh = oracle.sampler([g], HDDA, SKIP, CONSTANT, 0.1)
    for r in rays:
        nd, ed, _ = oracle.events(sd, r)
        nh, eh, _ = oracle.events(sh, r)
        assert nd == nh
        for a, b in zip(ed, eh):
            assert a[0] == b[0] and a[2] == b[2] and a[3] == b[3] and a[4] == b[4]


def test_sampling_known_answers(oracle):
    """test_sampling.cpp:63-84, 154-171"""
    full = Grid((4, 4, 4), (0.0, 0.0, 0.0), 1.0, np.full(8, 0xFF, np.uint8))
    ray = np.array([[-1.0, 0.5, 0.5, 1.0, 0.0, 0.0, 0.0, 100.0]])
    for an in (DDA, HDDA):
        for k in (BRANCH, SKIP):
            p = oracle.sample(oracle.sampler([full], an, k, CONSTANT, 0.25), ray)
            assert p.total == 16 and p.t_starts[0] == 1.25 and p.t_starts[-1] == 5.0
    empty = Grid((16, 16, 16), (0.0, 0.0, 0.0), 1.0, np.zeros(512, np.uint8))
    p = oracle.sample(oracle.sampler([empty], DDA, BRANCH, CONSTANT, 0.5),
                      np.array([[-1.0, 8.5, 8.5, 1.0, 0.0, 0.0, 0.0, 100.0]]))
    assert p.total == 0
    g = _unit128_block([16, 96], 56, 56)
    ray = np.array([[-1.0, 60.5, 60.5, 1.0, 0.0, 0.0, 0.0, 1000.0]])
    br = oracle.sample(oracle.sampler([g], HDDA, BRANCH, CONSTANT, 0.5), ray)
    sk = oracle.sample(oracle.sampler([g], HDDA, SKIP, CONSTANT, 0.5), ray)
    assert _eq64(br.t_starts, sk.t_starts) and br.total > 0
    assert sk.counters[0, 2] == 0
    assert sk.counters[0, 0] + sk.counters[0, 2] < br.counters[0, 0] + br.counters[0, 2]


def test_linear_schedule_gaps_non_decreasing(oracle):
    """test_sampling.cpp:173-189"""
    full = Grid((4, 4, 4), (0.0, 0.0, 0.0), 1.0, np.full(8, 0xFF, np.uint8))
    p = oracle.sample(oracle.sampler([full], DDA, SKIP, LINEAR, 0.01, 1.0 / 64),
                      np.array([[-1.0, 0.5, 0.5, 1.0, 0.0, 0.0, 0.0, 100.0]]))
    b = p.t_starts
    assert b.size > 3
    assert np.all(np.diff(b)[1:] >= np.diff(b)[:-1] - 1e-15)


def test_vdb_collapse_and_queries(oracle):
    """test_vdb_tree.cpp:32-129 and :218-254"""
    C = __import__("ctypes")
    empty = Grid((128, 128, 128), (-1.0, -1.0, -1.0), 2.0 / 128, np.zeros(128 ** 3 // 8, np.uint8))
    b = oracle.sog1(empty)
    assert len(b) == 4 + 4 + 12 + 24 + 8 + 4 + 13 and b[-1] == 0  # one empty root tile
    full = Grid(empty.res, empty.wmin, empty.voxel, np.full(empty.bits.size, 0xFF, np.uint8))
    assert oracle.sog1(full)[-1] == 1
    g = _unit128_block([0])
    sp = oracle.sparse(g)
    lvl, ext = C.c_int32(), C.c_int32()
    org = np.zeros(3, np.int32)
    occ = oracle.L.og_sparse_query(sp, np.array([3, 3, 3], np.int32), C.byref(lvl), org, C.byref(ext))
    assert occ == 1 and lvl.value == 1 and list(org) == [0, 0, 0] and ext.value == 8
    occ = oracle.L.og_sparse_query(sp, np.array([-3, 5, 5], np.int32), C.byref(lvl), org, C.byref(ext))
    assert occ == 0 and lvl.value == 3 and list(org) == [-128, 0, 0] and ext.value == 128


def test_oracle_vs_reference_randomized(oracle, reflib, P):
    """Oracle == reference on seeded random grids/rays, every variant (skipped without oracle/_ref)."""
    t = P.GridTransform.cube(32, (-1, -1, -1), 2.0)
    for seed in (1, 2):
        g = reflib.random_blocky_grid((32, 32, 32), (-1.0, -1.0, -1.0), 2.0 / 32, seed, 0.2, 0.03)
        rays = P.random_rays(t, 400, seed + 10)
        for an in (DDA, HDDA):
            for k in (BRANCH, SKIP):
                for sk, dt, gr in ((CONSTANT, 0.017, 0.0), (LINEAR, 0.011, 1.0 / 256)):
                    o = oracle.sample(oracle.sampler([g], an, k, sk, dt, gr), rays)
                    r = reflib.sampler([g], an, k, sk, dt, gr).sample(rays, skip=(o.status == 2))
                    assert np.array_equal(o.packed_info, r.packed_info)
                    assert _eq64(o.t_starts, r.t_starts) and _eq64(o.t_ends, r.t_ends)
                    assert np.array_equal(o.cells, r.cells) and np.array_equal(o.counters, r.counters)


def test_oracle_vs_reference_config_shapes(oracle, reflib, P):
    """The oracle pinned to the unmodified reference at the benchmark configurations' shapes
    (CPU, sub-sampled rays): 128^3 scenes of cfg2 on orbit-camera rays, the 4-level cfg3 cascade
    at 1297x840 (linear schedule, the spinning u == 0 column included and screened), and 512^3
    blobs with make_probe_rays (cfg4) -- every variant, outputs and counters bit for bit."""
    from oracle_bindings import CD

    def same(o, r, what):
        ok = o.status != 2
        assert np.array_equal(o.packed_info[ok, 1], r.packed_info[ok, 1]), what
        assert _eq64(o.t_starts, r.t_starts) and _eq64(o.t_ends, r.t_ends), what
        assert np.array_equal(o.cells, r.cells) and np.array_equal(o.levels, r.levels), what
        assert np.array_equal(o.counters[ok], r.counters[ok]), what

    cam = reflib.camera_rays((2.9, 1.4, -1.3), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, 800, 800)[::211]
    for kind, kw in (("shell", dict(seed=2, count=256)), ("blobs", dict(seed=3, count=24)),
                     ("sponge", dict(seed=1)), ("random", dict(seed=1, fraction=0.02))):
        g = reflib.scene(kind, 128, seed=kw["seed"], fraction=kw.get("fraction", 0.05), count=kw.get("count", 12))
        for an in (DDA, HDDA, CD):
            for k in (BRANCH, SKIP):
                o = oracle.sample(oracle.sampler([g], an, k, CONSTANT, 0.5 * g.voxel), cam)
                r = reflib.sampler([g], an, k, CONSTANT, 0.5 * g.voxel).sample(cam, skip=(o.status == 2))
                same(o, r, f"{kind} an={an} k={k}")
    lv = reflib.cascade("blobs", 4, 128, seed=1)
    rays = reflib.camera_rays((1.9, 1.4, 2.3), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, 1297, 840)
    sub = np.concatenate([rays[::97], rays[648::1297]])  # a strided sample + the u == 0 column
    for an in (DDA, HDDA):
        o = oracle.sample(oracle.sampler(lv, an, SKIP, LINEAR, 0.5 * lv[0].voxel, 1.0 / 256, cascade=True), sub)
        r = reflib.sampler(lv, an, SKIP, LINEAR, 0.5 * lv[0].voxel, 1.0 / 256, cascade=True).sample(
            sub, skip=(o.status == 2))
        same(o, r, f"cascade an={an}")
    g = reflib.scene("blobs", 512, seed=1)
    probe = reflib.probe_rays(g, 3000, 1000)
    for an in (DDA, HDDA):
        o = oracle.sample(oracle.sampler([g], an, SKIP, CONSTANT, 0.5 * g.voxel), probe)
        r = reflib.sampler([g], an, SKIP, CONSTANT, 0.5 * g.voxel).sample(probe, skip=(o.status == 2))
        same(o, r, f"512^3 an={an}")
