"""Out-of-bounds write guards for the sampling kernels (pass 1, scan, pass 2 gather / tail /
cold write) and the traverse writer.

Every output array lives inside a larger allocation with a guard band of sentinel bytes on both
sides. After each call the guards must still hold the sentinel, and the outputs between them
must equal the oracle's bit for bit. The calls cover DDA / HDDA / CD, skip / branch, constant /
linear schedules, a cascade, slab overflow (SOGK_SLAB=1: most rays finish in tail_kernel), the
cold write (no matching count), and outputs off their natural alignment. This stands in for
compute-sanitizer's memcheck, which is not available on the GPU pool. A misaligned packed_info
(the kernels access its {offset, count} pairs as 16-byte units) is refused, not faulted.
"""
import numpy as np
import pytest
import torch

from oracle_bindings import BRANCH, CD, DDA, HDDA, SKIP
from parity_util import bits64, gpu_grids, host_grid, oracle_sample, scene_grid

pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes on each side
SENTINEL = 0xA5


def _guarded(n, dtype, offset, dev):
    """A tensor of n elements that starts GUARD + offset elements into a sentinel-filled block."""
    item = torch.empty(0, dtype=dtype).element_size()
    lead = GUARD // item + offset
    raw = torch.full((lead + n + GUARD // item,), 0, dtype=dtype, device=dev)
    raw.view(torch.uint8).fill_(SENTINEL)
    return raw, raw[lead:lead + n], lead


def _guards_intact(raw, lead, n, what):
    b = raw.view(torch.uint8).cpu().numpy()
    item = raw.element_size()
    head, tail = b[:lead * item], b[(lead + n) * item:]
    assert (head == SENTINEL).all(), f"{what}: write before the buffer"
    assert (tail == SENTINEL).all(), f"{what}: write past the buffer"


def _sample_guarded(P, levels, an, k, sched, rays, cascade, offset, cold):
    dev = torch.device("cuda")
    grids = gpu_grids(P, levels, an)
    s = P.Sampler(grids, an, k, sched, cascade=cascade)
    d = torch.from_numpy(np.ascontiguousarray(rays, np.float64).reshape(-1, 8)).to(dev)
    n = d.shape[0]
    praw, packed, plead = _guarded(2 * n, torch.int64, 2 * offset, dev)  # {offset, count} pairs: 16-byte aligned
    sraw, status, slead = _guarded(n, torch.uint8, offset, dev)
    craw, counters, clead = _guarded(3 * n, torch.int32, offset, dev)
    packed = packed.view(n, 2)
    packed_c, stats = s.count(d, status, counters.view(n, 3), packed_info=packed)
    total = int(stats.cpu()[P.STAT_TOTAL_SAMPLES])
    outs = {}
    raws = []
    for key, dt in (("t_starts", torch.float64), ("t_ends", torch.float64), ("ray_indices", torch.int32),
                    ("cells", torch.int32), ("levels", torch.uint8)):
        raw, view, lead = _guarded(total, dt, offset, dev)
        outs[key] = view
        raws.append((key, raw, lead, total))
    if cold:  # a packed_info copy the count did not fill: the exact cold path (write_kernel)
        packed_w = packed.clone()
    else:
        packed_w = packed
    s.write(d, packed_w, total, out=outs)
    torch.cuda.synchronize()
    what = f"an={an} k={k} sched={sched.kind} cascade={cascade} offset={offset} cold={cold}"
    _guards_intact(praw, plead, 2 * n, what + " packed_info")
    _guards_intact(sraw, slead, n, what + " status")
    _guards_intact(craw, clead, 3 * n, what + " counters")
    for key, raw, lead, m in raws:
        _guards_intact(raw, lead, m, f"{what} {key}")
    return packed.cpu().numpy(), {k: v.cpu().numpy() for k, v in outs.items()}, counters.view(n, 3).cpu().numpy()


def _check(got, want, what):
    pi, o, ctr = got
    assert np.array_equal(pi, want.packed_info), what
    assert np.array_equal(bits64(o["t_starts"]), bits64(want.t_starts)), what
    assert np.array_equal(bits64(o["t_ends"]), bits64(want.t_ends)), what
    assert np.array_equal(o["ray_indices"], want.ray_indices), what
    assert np.array_equal(o["cells"].view(np.uint32), want.cells), what
    assert np.array_equal(o["levels"], want.levels), what
    assert np.array_equal(ctr, want.counters), what


@pytest.mark.parametrize("slab", [None, "1"])
@pytest.mark.parametrize("offset", [0, 1])
def test_sampling_writes_stay_in_bounds(P, oracle, monkeypatch, slab, offset):
    if slab is not None:
        monkeypatch.setenv("SOGK_SLAB", slab)
    g = scene_grid(P, "blobs", 48, seed=3, count=10)
    rays = np.asarray(P.random_rays(P.GridTransform(g.res, g.wmin, g.voxel), 1500, 9), np.float64)
    for an in (DDA, HDDA, CD):
        for k in (SKIP, BRANCH):
            for sched in (P.StepSchedule.constant(0.5 * g.voxel), P.StepSchedule.linear(0.4 * g.voxel, 1.0 / 64)):
                for cold in (False, True):
                    got = _sample_guarded(P, [g], an, k, sched, rays, False, offset, cold)
                    want = oracle_sample(oracle, [g], an, k, sched, rays)
                    _check(got, want, f"an={an} k={k} sched={sched.kind} cold={cold}")


def test_cascade_writes_stay_in_bounds(P, oracle):
    base = P.GridTransform.cube(32, (-1.0, -1.0, -1.0), 2.0)
    levels = []
    for b in range(3):  # concentric levels at (-s, -s, -s), the shape of test_sampling.cpp:274-293
        sc = float(1 << b)
        t = P.GridTransform(base.resolution, (-sc, -sc, -sc), base.voxel_size * sc)
        levels.append(host_grid(P, t, P.random_blocky_grid(t, 71 + b, 0.1, 0.01)))
    rays = np.asarray(P.random_rays(P.GridTransform(levels[-1].res, levels[-1].wmin, levels[-1].voxel),
                                    1200, 4), np.float64)
    sched = P.StepSchedule.linear(0.5 * base.voxel_size, 1.0 / 128)
    for an in (DDA, HDDA):
        for k in (SKIP, BRANCH):
            got = _sample_guarded(P, levels, an, k, sched, rays, True, 1, False)
            want = oracle_sample(oracle, levels, an, k, sched, rays, cascade=True)
            _check(got, want, f"cascade an={an} k={k}")


def test_traverse_writes_stay_in_bounds(P):
    dev = torch.device("cuda")
    g = scene_grid(P, "shell", 48, seed=1)
    rays = np.asarray(P.random_rays(P.GridTransform(g.res, g.wmin, g.voxel), 800, 2), np.float64)
    d = torch.from_numpy(rays.reshape(-1, 8)).to(dev)
    n = d.shape[0]
    for an in (DDA, HDDA, CD):
        s = P.Sampler(gpu_grids(P, [g], an), an, SKIP, P.StepSchedule.constant(0.5 * g.voxel))
        iraw, info, ilead = _guarded(2 * n, torch.int64, 2, dev)
        st = torch.empty(P.STATS_LEN, dtype=torch.int64, device=dev)
        P._check(P.lib.sogk_traverse_count(s._h, d.data_ptr(), n, info.data_ptr(), st.data_ptr(), None, None, None),
                 "traverse count")
        total = int(st.cpu()[P.STAT_TOTAL_SAMPLES])
        ev_bytes = 40
        eraw, ev, elead = _guarded(total * ev_bytes, torch.uint8, 8, dev)
        P._check(P.lib.sogk_traverse_write(s._h, d.data_ptr(), n, info.data_ptr(), ev.data_ptr(), None),
                 "traverse write")
        torch.cuda.synchronize()
        _guards_intact(iraw, ilead, 2 * n, f"an={an} event_info")
        _guards_intact(eraw, elead, total * ev_bytes, f"an={an} events")
        counts = info.view(n, 2).cpu().numpy()[:, 1]
        assert counts.sum() == total and total > 0


def test_misaligned_pair_buffers_are_refused(P):
    """The {offset, count} pairs and the rays are 16-byte accesses: a misaligned base is an
    argument error (the context stays usable), not a kernel fault."""
    dev = torch.device("cuda")
    g = scene_grid(P, "blobs", 32, seed=1)
    rays = np.asarray(P.random_rays(P.GridTransform(g.res, g.wmin, g.voxel), 64, 3), np.float64)
    d = torch.from_numpy(rays.reshape(-1, 8)).to(dev)
    s = P.Sampler(gpu_grids(P, [g], HDDA), HDDA, SKIP, P.StepSchedule.constant(0.5 * g.voxel))
    raw = torch.zeros(2 * 64 + 1, dtype=torch.int64, device=dev)
    with pytest.raises(ValueError, match="16-byte aligned"):
        s.count(d, packed_info=raw[1:].view(64, 2))
    rraw = torch.zeros(64 * 8 + 1, dtype=torch.float64, device=dev)
    rraw[1:] = d.reshape(-1)
    with pytest.raises(ValueError, match="16-byte aligned"):
        s.count(rraw[1:].view(64, 8))
    out = s.sample(d)  # still usable
    torch.cuda.synchronize()
    assert out.packed_info.shape[0] == 64
