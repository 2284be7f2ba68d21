"""GPU robustness: stream ordering of grid builds, the pass-1 -> pass-2 handshake token,
host-thread safety of one sampler, the resume-record packing of very long rays, the
render scratch paths and the argument guards of the C-ABI (include/sogk.h "Limits")."""
import ctypes as C
import threading

import numpy as np
import pytest
import torch

from oracle_bindings import DDA, HDDA, SKIP, BRANCH, Grid
from parity_util import (assert_packed_equal, bits64, host_grid, oracle_sample, scene_grid,
                         to_packed)

pytestmark = pytest.mark.gpu


def test_grid_built_on_side_stream_sampled_on_another(P, oracle):
    """VDB and distance builds are stream-ordered (pool storage + build event); a sampler
    used on a different non-blocking stream, with no host synchronisation, must see the
    finished grid (every launch waits on the levels' build events)."""
    g = scene_grid(P, "shell", 128, seed=1)
    t = P.GridTransform(g.res, g.wmin, g.voxel)
    rays = P.random_rays(t, 20000, seed=3)
    sched = P.StepSchedule.constant(0.5 * g.voxel)
    want = oracle_sample(oracle, [g], HDDA, SKIP, sched, rays)
    d = torch.from_numpy(rays).cuda()
    dense = P.DenseGrid(t, g.bits)
    torch.cuda.synchronize()
    for _ in range(3):
        a, b = torch.cuda.Stream(), torch.cuda.Stream()
        vdb = P.build_sparse(dense, stream=a)  # no sync after this
        s = P.Sampler([vdb], HDDA, SKIP, sched)
        out = s.sample(d, stream=b)
        assert_packed_equal(to_packed(out), want, "side-stream build")


def test_token_handshake_buffer_rewritten_in_place(P, oracle):
    """count(A) on stream X, the ray buffer overwritten with B and counted on stream Y into the
    same packed_info, then write on X: the write must not use X's slabs of A (pointer-keyed
    matching would); it takes the exact cold path and returns B's samples."""
    g = scene_grid(P, "blobs", 64, seed=2)
    t = P.GridTransform(g.res, g.wmin, g.voxel)
    ra = P.random_rays(t, 5000, seed=1)
    rb = P.random_rays(t, 5000, seed=2)
    sched = P.StepSchedule.constant(0.5 * g.voxel)
    s = P.Sampler([P.build_sparse(P.DenseGrid(t, g.bits))], HDDA, SKIP, sched)
    d = torch.from_numpy(ra).cuda()
    x, y = torch.cuda.Stream(), torch.cuda.Stream()
    packed = torch.empty((5000, 2), dtype=torch.int64, device="cuda")
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    x.wait_stream(torch.cuda.current_stream())
    s.count(d, stream=x, packed_info=packed, stats=stats)
    x.synchronize()
    d.copy_(torch.from_numpy(rb))
    torch.cuda.synchronize()
    y.wait_stream(torch.cuda.current_stream())
    s.count(d, stream=y, packed_info=packed, stats=stats)
    y.synchronize()
    total = int(stats[0].item())
    with torch.cuda.stream(x):
        ts, te, ri, ce, lv = s.write(d, packed, total, stream=x)
    x.synchronize()
    want = oracle_sample(oracle, [g], HDDA, SKIP, sched, rb)
    assert np.array_equal(packed.cpu().numpy(), want.packed_info)
    assert np.array_equal(bits64(ts.cpu().numpy()), bits64(want.t_starts))
    assert np.array_equal(ce.cpu().numpy().view(np.uint32), want.cells)


def test_one_sampler_many_host_threads(P, oracle):
    """make_sampler's function is called from render_frame's worker threads at once
    (bench.hpp:446-454): concurrent sogk_sample_host calls on one sampler are serialised by
    the sampler's lock and each returns its own rays' samples."""
    g = scene_grid(P, "shell", 64, seed=1)
    t = P.GridTransform(g.res, g.wmin, g.voxel)
    sched = P.StepSchedule.constant(0.5 * g.voxel)
    s = P.Sampler([P.build_sparse(P.DenseGrid(t, g.bits))], HDDA, SKIP, sched)
    batches = [P.random_rays(t, 3000 + 17 * i, seed=40 + i) for i in range(8)]
    outs = [None] * len(batches)
    errs = []

    def work(i):
        try:
            for _ in range(3):
                outs[i] = s.sample_host(batches[i])
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(batches))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for i, r in enumerate(batches):
        assert_packed_equal(to_packed(outs[i]), oracle_sample(oracle, [g], HDDA, SKIP, sched, r), f"thread {i}")


def test_resume_after_2_pow_23_samples(P, oracle, monkeypatch):
    """A ray whose first run leaves more than 2^23 samples in its slab before the next run
    overflows it: the resume record packs that count into bits 8..31 of its tag, unsigned
    (a signed shift made it negative and tail_kernel wrote before the ray's range)."""
    t = P.GridTransform((4, 1, 1), (0.0, 0.0, 0.0), 1.0)
    bits = np.array([0b0101], np.uint8)  # voxels 0 and 2 occupied
    g = host_grid(P, t, bits)
    dt = 1.0 / float((1 << 23) + 4099)
    sched = P.StepSchedule.constant(dt)
    ray = np.array([[-0.5, 0.5, 0.5, 1.0, 0.0, 0.0, 0.0, 100.0]])
    want = oracle_sample(oracle, [g], DDA, SKIP, sched, ray)
    assert want.total > (1 << 24)
    for an in (DDA, HDDA):
        grids = [P.DenseGrid(t, g.bits)]
        if an == HDDA:
            grids = [P.build_sparse(grids[0])]
        s = P.Sampler(grids, an, SKIP, sched)
        out = s.sample(torch.from_numpy(ray).cuda())
        got = to_packed(out)
        assert int(out.stats[6]) == 1, "the second run must overflow the slab"
        assert np.array_equal(got.packed_info, want.packed_info)
        assert np.array_equal(bits64(got.t_starts), bits64(want.t_starts))
        assert np.array_equal(bits64(got.t_ends), bits64(want.t_ends))


def test_render_bound_path_equals_sync_path(P, monkeypatch):
    """sogk_render_camera sizes its sample scratch from the camera's bound (no host round
    trip) when that fits, else reads the total back; both give the same frame bit for bit,
    and repeated frames are identical."""
    t = P.GridTransform.cube(64, (-1.0, -1.0, -1.0), 2.0)
    g = scene_grid(P, "shell", 64, seed=1)
    scene = P.analytic_scene("shell", t, seed=1)
    cam = P.Camera((1.9, 1.4, 2.3), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, 120, 90)
    sched = P.StepSchedule.constant(0.5 * g.voxel)
    s = P.Sampler([P.build_sparse(P.DenseGrid(t, g.bits))], HDDA, SKIP, sched)
    f1 = P.render_frame(s, scene, cam)
    f2 = P.render_frame(s, scene, cam)
    monkeypatch.setenv("SOGK_RENDER_SYNC", "1")
    f3 = P.render_frame(s, scene, cam)
    r1, r2, r3 = (f.result.cpu().numpy().view(np.uint64) for f in (f1, f2, f3))
    assert np.array_equal(r1, r2) and np.array_equal(r1, r3)
    assert (f1.lookups, f1.steps, f1.samples) == (f3.lookups, f3.steps, f3.samples)


def test_argument_guards(P):
    g = scene_grid(P, "blobs", 32, seed=1)
    t = P.GridTransform(g.res, g.wmin, g.voxel)
    sched = P.StepSchedule.constant(0.5 * g.voxel)
    s = P.Sampler([P.DenseGrid(t, g.bits)], DDA, BRANCH, sched)
    d = torch.from_numpy(P.random_rays(t, 100, seed=1)).cuda()
    packed, stats = s.count(d)
    total = int(stats[0].item())
    with pytest.raises(ValueError, match="INT32_MAX"):
        s.write(d, packed, max(total, 1), ray_index_base=(1 << 31) - 50)
    # n >= 2^32 is refused before any buffer is touched
    st = P.lib.sogk_sample_count(s._h, d.data_ptr(), 1 << 32, packed.data_ptr(), stats.data_ptr(),
                                 None, None, None)
    assert st == P.INVALID_ARG
    # cells pack 10 bits per axis: refused above 1024 voxels
    tw = P.GridTransform((1100, 8, 8), (0.0, 0.0, 0.0), 1.0)
    sw = P.Sampler([P.DenseGrid(tw, np.zeros(tw.payload_bytes(), np.uint8))], DDA, SKIP, sched)
    ray = torch.tensor([[-1.0, 4.5, 4.5, 1.0, 0.0, 0.0, 0.0, 2000.0]], dtype=torch.float64, device="cuda")
    pk, _ = sw.count(ray)
    with pytest.raises(ValueError, match="1024"):
        sw.write(ray, pk, 1, cells=True)
    sw.write(ray, pk, 1, cells=False)  # without cells it is fine
