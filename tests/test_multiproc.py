"""Multi-process (world_size 2, gloo on CPU) coverage of the sharded path: the grid
payload is broadcast once from rank 0, each rank samples its contiguous ray shard with
globally numbered ray_indices, and the gathered result is identical to one process
(the reference's thread-count invariance, test_scene_bench.cpp:232-250, across ranks).
The CPU oracle stands in for the GPU kernels, which the -m gpu tests pin to it."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2404_10272_b200 as P
    from paper_2404_10272_b200.shard import broadcast_payload, shard_range, view_of
    from oracle_bindings import HDDA, SKIP, Grid, Oracle

    t = P.GridTransform.cube(48, (-1.0, -1.0, -1.0), 2.0)
    bits = torch.zeros(t.payload_bytes(), dtype=torch.uint8)
    if rank == 0:
        bits = torch.from_numpy(P.generate_scene("shell", t, seed=1)[0])
    broadcast_payload(bits)
    g = Grid(t.resolution, t.world_min, t.voxel_size, bits.numpy())
    rays = P.Camera((1.9, 1.4, 2.3), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, 61, 43).rays()
    a, b = shard_range(rays.shape[0], world, rank)
    O = Oracle()
    s = O.sampler([g], HDDA, SKIP, 0, 0.5 * t.voxel_size)
    p = O.sample(s, rays[a:b], ray_index_base=a)
    parts = [None] * world
    dist.all_gather_object(parts, (p.packed_info[:, 1], p.t_starts, p.ray_indices, p.cells))
    views = [None] * world
    dist.all_gather_object(views, [view_of(k, rank, world) for k in range(5)])
    if rank == 0:
        full = O.sample(s, rays)
        q.put(dict(
            counts=np.array_equal(np.concatenate([x[0] for x in parts]), full.packed_info[:, 1]),
            t=np.array_equal(np.concatenate([x[1] for x in parts]).view(np.uint64), full.t_starts.view(np.uint64)),
            ri=np.array_equal(np.concatenate([x[2] for x in parts]), full.ray_indices),
            cells=np.array_equal(np.concatenate([x[3] for x in parts]), full.cells),
            views_disjoint=len({v for vs in views for v in vs}) == 5 * world,
        ))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharding_is_rank_count_invariant():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res


def test_shard_ranges_cover_exactly():
    from paper_2404_10272_b200.shard import shard_range

    for n in (0, 1, 7, 640000, 1089480):
        for w in (1, 2, 3, 4, 8):
            rs = [shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
