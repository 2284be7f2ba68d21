"""The compositing consumer's checkers (render.hpp), CPU only: the host AnalyticScene generator
and the oracle's composite_detailed pinned to the unmodified reference, plus the reference
unit suite's known answers (proj/tests/unit/test_render.cpp)."""
import math

import numpy as np
import pytest

from oracle_bindings import CONSTANT, HDDA, LINEAR, SKIP, Grid


def _as16(prims):
    return np.array([[p.shape, *p.center, p.radius, *p.lo, *p.hi, p.density, *p.color, 0.0]
                     for p in prims], np.float64)


@pytest.mark.parametrize("kind", ["blobs", "shell", "sponge", "random"])
@pytest.mark.parametrize("seed", [1, 7])
def test_analytic_scene_matches_reference(P, reflib, kind, seed):
    t = P.GridTransform.cube(128, (-1.0, -1.0, -1.0), 2.0)
    mine = P.analytic_scene(kind, t, seed=seed, count=24)
    ref, bg = reflib.scene_primitives(kind, 128, seed=seed, count=24)
    assert np.array_equal(_as16(mine.primitives).view(np.uint64), ref.view(np.uint64))
    assert np.array_equal(np.asarray(mine.background), bg)


def test_composite_known_answers(P, oracle):
    """test_render.cpp:33-53 and :88-99."""
    ray = [0, 0, 0, 1, 0, 0, 0.0, 10.0]
    c = oracle.composite(ray, [], [], (0.2, 0.4, 0.6), CONSTANT, 0.1)
    assert list(c[:3]) == [0.2, 0.4, 0.6]  # no samples yields the background
    prims = [P.Primitive.sphere((5, 0, 0), 1.0, 250.0, (0.3, 0.7, 0.9))]
    c = oracle.composite(ray, [5.0], prims, (1, 0, 0), CONSTANT, 0.1)
    assert abs(c[0] - 0.3) < 1e-8 and abs(c[1] - 0.7) < 1e-8 and abs(c[2] - 0.9) < 1e-8
    rng = np.random.default_rng(123)
    prims = [P.Primitive.sphere(rng.uniform(-1, 1, 3), rng.uniform(0.1, 0.5), rng.uniform(0.5, 8.0),
                                (0.5, 0.5, 0.5)) for _ in range(6)]
    samples = np.arange(0.5, 4.0, 0.01)
    t = P.GridTransform.cube(8, (-1, -1, -1), 2.0)
    for r in P.random_rays(t, 200, seed=5):
        c = oracle.composite(r, samples, prims, (0.1, 0.1, 0.1), CONSTANT, 0.01)
        assert abs(c[3] + c[4] - 1.0) <= 1e-12  # weight sum plus transmittance is one


def test_slab_quadrature_first_order(P, oracle):
    """test_render.cpp:58-78: ladder quadrature through a slab converges at first order."""
    sigma, x0 = 0.9, 2.0137
    x1 = x0 + math.sqrt(3.0)
    exact = 1.0 - math.exp(-sigma * (x1 - x0))
    prims = [P.Primitive.box((x0, -10, -10), (x1, 10, 10), sigma, (1.0, 1.0, 1.0))]
    rng = np.random.default_rng(99)

    def err(dt):
        s = 0.0
        for _ in range(64):
            ph = rng.uniform(0.0, dt)
            ts, t = [], dt
            while t <= 100.0:
                if x0 <= ph + t < x1:
                    ts.append(t)
                t += dt
            s += abs(oracle.composite([ph, 0, 0, 1, 0, 0, 0.0, 100.0], ts, prims, (0, 0, 0),
                                      CONSTANT, dt)[3] - exact)
        return s / 64

    e1, e2 = err(1.0 / 32.0), err(1.0 / 64.0)
    assert 0.6 < e1 / e2 < 6.0 and e2 < e1


@pytest.mark.parametrize("kind,sched", [("shell", CONSTANT), ("blobs", LINEAR), ("sponge", CONSTANT)])
def test_oracle_composite_equals_reference(P, oracle, reflib, kind, sched):
    """og_composite == the reference's composite_detailed bit for bit on real sample buffers."""
    t = P.GridTransform.cube(32, (-1.0, -1.0, -1.0), 2.0)
    bits, _ = P.generate_scene(kind, t, seed=2)
    g = Grid(tuple(t.resolution), tuple(t.world_min), t.voxel_size, bits)
    scene = P.analytic_scene(kind, t, seed=2)
    ref16 = _as16(scene.primitives)
    dt0, growth = 0.5 * t.voxel_size, 1.0 / 128.0
    s = oracle.sampler([g], HDDA, SKIP, sched, dt0, growth)
    rays = P.random_rays(t, 300, seed=4)
    pk = oracle.sample(s, rays)
    for i in range(rays.shape[0]):
        o, n = pk.packed_info[i]
        smp = pk.t_starts[o:o + n]
        a = oracle.composite(rays[i], smp, scene.primitives, scene.background, sched, dt0, growth)
        b = reflib.composite(rays[i], smp, ref16, scene.background, sched, dt0, growth)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), i
    # set_pixel / psnr agree with the Python mirror
    img_a = np.array([oracle.set_pixel(c) for c in [(0.5, 1.2, -0.1), (0.0019, 0.998, 0.5)]])
    assert img_a.tolist() == [[128, 255, 0], [0, 254, 128]]
    assert P.psnr(img_a, img_a) == 99.0
