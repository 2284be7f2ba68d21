"""GPU compositing consumer (render.hpp) vs the CPU oracle and the unmodified reference.

Tolerance: the compositor calls exp(); CUDA's double exp is within 1 ulp but not always the
correctly rounded glibc value, so colors / weight sums / transmittances are compared at
1e-12 relative (plus 1e-15 absolute), 8-bit pixels within 1 level and the reference's own
acceptance gate (render_frame PSNR >= 40 dB, acceptance_main.cpp:143-170).  Frame counters
(lookups, steps, samples) are exact.
"""
import numpy as np
import pytest
import torch

from oracle_bindings import BRANCH, CONSTANT, DDA, HDDA, LINEAR, SKIP
from parity_util import VARIANTS, gpu_grids, host_grid, oracle_sample, scene_grid

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-12, 1e-15


def _bench_camera(P, w, h):
    return P.Camera((1.9, 1.4, 2.3), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, w, h)


@pytest.mark.parametrize("kind", ["shell", "blobs", "sponge"])
def test_composite_matches_oracle(P, oracle, kind):
    t = P.GridTransform.cube(64, (-1.0, -1.0, -1.0), 2.0)
    g = scene_grid(P, kind, 64, seed=2)
    scene = P.analytic_scene(kind, t, seed=2)
    rays = _bench_camera(P, 96, 72).rays()
    for sched in (P.StepSchedule.constant(0.5 * g.voxel), P.StepSchedule.linear(0.5 * g.voxel, 1.0 / 128)):
        s = P.Sampler(gpu_grids(P, [g], HDDA), HDDA, SKIP, sched)
        d = torch.from_numpy(rays).cuda()
        out = s.sample(d)
        res, rgb = P.composite(s, scene, d, out.packed_info, out.t_starts)
        res, rgb = res.cpu().numpy(), rgb.cpu().numpy()
        pk = out.packed_info.cpu().numpy()
        ts = out.t_starts.cpu().numpy()
        for i in range(rays.shape[0]):
            o, n = pk[i]
            want = oracle.composite(rays[i], ts[o:o + n], scene.primitives, scene.background,
                                    sched.kind, sched.dt0, sched.growth)
            np.testing.assert_allclose(res[i], want, rtol=RTOL, atol=ATOL)
            assert np.abs(rgb[i].astype(int) - oracle.set_pixel(want[:3]).astype(int)).max() <= 1


def test_fused_render_equals_composite_of_packed(P):
    """render_frame's fused kernel == sample_count/write + composite, bit for bit (same device
    arithmetic), for every variant and both schedules."""
    t = P.GridTransform.cube(64, (-1.0, -1.0, -1.0), 2.0)
    g = scene_grid(P, "shell", 64, seed=1)
    scene = P.analytic_scene("shell", t, seed=1)
    cam = _bench_camera(P, 80, 60)
    for sched in (P.StepSchedule.constant(0.5 * g.voxel), P.StepSchedule.linear(0.011, 1.0 / 256)):
        for an, k in VARIANTS:
            s = P.Sampler(gpu_grids(P, [g], an), an, k, sched)
            f = P.render_frame(s, scene, cam)
            d = cam.rays_device()
            out = s.sample(d)
            res, rgb = P.composite(s, scene, d, out.packed_info, out.t_starts)
            assert np.array_equal(f.result.cpu().numpy().view(np.uint64), res.cpu().numpy().view(np.uint64))
            assert np.array_equal(f.image.reshape(-1, 3), rgb.cpu().numpy())
            assert f.samples == out.total
            c = out.counters.cpu().numpy().astype(np.int64)
            assert f.lookups == int(c[:, 0].sum() + c[:, 2].sum()) and f.steps == int(c[:, 1].sum())


@pytest.mark.parametrize("kind,seed,fraction", [("blobs", 1, 0.0), ("shell", 3, 0.0), ("sponge", 4, 0.0),
                                                ("random", 5, 0.03)])
def test_render_frame_vs_reference(P, reflib, kind, seed, fraction):
    """The acceptance gate's scenes (acceptance_main.cpp:146-170) at 160x120: the GPU frame of
    every variant against the reference's render_frame of the same variant (PSNR >= 40, in
    practice 99 = identical) and against its FrameResult counters (exact)."""
    t = P.GridTransform.cube(128, (-1.0, -1.0, -1.0), 2.0)
    bits, _ = P.generate_scene(kind, t, seed=seed, fraction=fraction if fraction > 0 else 0.05)
    g = host_grid(P, t, bits)
    scene = P.analytic_scene(kind, t, seed=seed)
    sched = P.StepSchedule.constant(0.5 * t.voxel_size)
    cam = _bench_camera(P, 160, 120)
    for an, k in ((DDA, BRANCH), (HDDA, SKIP), (HDDA, BRANCH)):
        img_ref, lk, st, smp = reflib.render_frame(kind, seed, fraction, 128, 1, 0, 160, 120,
                                                   grid=1 if an == HDDA else 0, analyzer=an, kernel=k)
        f = P.render_frame(P.Sampler(gpu_grids(P, [g], an), an, k, sched), scene, cam)
        p = P.psnr(f.image, img_ref)
        assert p >= 40.0, (kind, an, k, p)
        assert (f.lookups, f.steps, f.samples) == (lk, st, smp), (kind, an, k)
