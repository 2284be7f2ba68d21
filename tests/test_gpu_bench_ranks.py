"""bench.py's multi-rank path executed on one device: two ranks (torchrun, gloo backend on
CUDA tensors) run the grid broadcast, the contiguous ray shards with global ray_indices
(SURVEY §8e), the barriers and the max-over-ranks all_reduce, and the concatenation of the
ranks' GPU outputs equals the single-rank run bit for bit (the reference's thread-count
invariance, test_scene_bench.cpp:232-250, across ranks)."""
import glob
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(tmp, world, cfg):
    args = ["bench.py", "--config", cfg, "--steps", "2", "--warmup", "3", "--no-e2e", "--no-render",
            "--no-cpu-baseline", "--variants", "hdda_skip", "--dump", str(tmp)]
    if world == 1:
        cmd = [sys.executable] + args
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args + ["--backend", "gloo",
                                                                                     "--gpus", str(world)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return r.stdout


@pytest.mark.parametrize("cfg", ["cfg1", "cfg3"])
def test_two_ranks_concatenate_to_one(tmp_path, cfg):
    import json

    one = _run(tmp_path / "w1", 1, cfg)
    two = _run(tmp_path / "w2", 2, cfg)
    l2 = json.loads(two.strip().splitlines()[-1])
    assert l2["n_gpus"] == 2 and l2["scaling"] == "strong"
    a = np.load(tmp_path / "w1" / "rank0_obj0.npz")
    parts = [np.load(tmp_path / "w2" / f"rank{r}_obj0.npz") for r in range(2)]
    assert int(parts[0]["first"]) == 0 and int(parts[1]["first"]) == a["packed_info"].shape[0] - parts[1]["packed_info"].shape[0]
    for key in ("t_starts", "t_ends", "ray_indices", "cells", "status"):
        cat = np.concatenate([p[key] for p in parts])
        assert np.array_equal(cat.view(np.uint8), a[key].view(np.uint8)), key
    cnt = np.concatenate([p["packed_info"][:, 1] for p in parts])
    assert np.array_equal(cnt, a["packed_info"][:, 1])


def test_two_ranks_default_config_full_line(tmp_path):
    """The driver's scaling run: bench.py's default config (cfg2, views per rank, weak scaling)
    with every leg (e2e through sogk_sample_host, render) under two ranks; rank 0 prints one
    JSON line with the whole job's rays (two ranks' views)."""
    import json

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--backend", "gloo", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["rays_per_step"] == 2 * 8 * 800 * 800
    assert d["e2e"]["value"] > 0 and d["render"] is not None
    assert d["value"] > 0 and d["gpu_launches"] > 0
