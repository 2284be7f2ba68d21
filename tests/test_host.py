"""Host-side checks that need no GPU: the C-ABI library loads and exports every
symbol include/sogk.h declares, the host input generators reproduce the reference
generators bit for bit, and the API validates like the reference."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def _decls():
    src = open(os.path.join(ROOT, "include", "sogk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sogk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(P):
    names = _decls()
    assert len(names) >= 30
    lib = ctypes.CDLL(P.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert P.lib.sogk_abi_version() == 1
    assert b"sm_100a" in P.lib.sogk_version()


def test_kernels_are_sm100a_cubins(P):
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_scene_generators_match_reference_golden(P):
    g = np.load(GOLD)
    kinds = ["blobs", "shell", "sponge", "random"]
    for i in range(5):
        kind, res, seed, count = (int(x) for x in g[f"scene{i}_meta"])
        t = P.GridTransform.cube(res, (-1.0, -1.0, -1.0), 2.0)
        bits, _ = P.generate_scene(kinds[kind], t, seed=seed, fraction=float(g[f"scene{i}_frac"]), count=count)
        assert np.array_equal(bits, g[f"scene{i}_bits"]), i
    for i in range(2):
        res = tuple(int(x) for x in g[f"blocky{i}_res"])
        seed, bf, nf = g[f"blocky{i}_args"]
        t = P.GridTransform(res, (-1.0, -1.0, -1.0), 2.0 / res[0])
        assert np.array_equal(P.random_blocky_grid(t, int(seed), bf, nf), g[f"blocky{i}_bits"]), i
    for b in range(4):
        pass
    lv = P.build_dense_cascade("blobs", P.GridTransform.cube(32, (-1, -1, -1), 2.0), 4, seed=1)
    for b, (t, bits) in enumerate(lv):
        assert np.array_equal(bits, g[f"casc{b}_bits"])
        assert t.world_min == tuple(g[f"casc{b}_wmin"]) and t.voxel_size == float(g[f"casc{b}_voxel"])


def test_ray_generators_match_reference_golden(P):
    g = np.load(GOLD)
    t = P.GridTransform.cube(32, (-1.0, -1.0, -1.0), 2.0)
    u = lambda a: np.ascontiguousarray(a).view(np.uint64)  # noqa: E731
    assert np.array_equal(u(P.random_rays(t, 200, 7)), u(g["rays_random"]))
    assert np.array_equal(u(P.make_probe_rays(t, 200, 11)), u(g["rays_probe"]))
    cam = P.Camera((1.9, 1.4, 2.3), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, 21, 15)
    assert np.array_equal(u(cam.rays()), u(g["rays_camera"]))


def test_generators_vs_reference_randomized(P, reflib):
    for kind in ("blobs", "shell", "sponge", "random"):
        for res in (24, 64):
            t = P.GridTransform.cube(res, (-1.0, -1.0, -1.0), 2.0)
            bits, occ = P.generate_scene(kind, t, seed=5, fraction=0.07, count=9)
            assert np.array_equal(bits, reflib.scene(kind, res, seed=5, fraction=0.07, count=9).bits)
    for (w, h) in ((1297, 840), (64, 48)):
        cam = P.Camera((1.9, 1.4, 2.3), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, w, h)
        a, b = cam.rays(), reflib.camera_rays(width=w, height=h)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_api_validation_like_the_reference(P):
    with pytest.raises(ValueError):
        P.GridTransform((0, 4, 4), (0, 0, 0), 1.0)       # grid.hpp:26-27
    with pytest.raises(ValueError):
        P.GridTransform((4, 4, 4), (0, 0, 0), 0.0)       # grid.hpp:28-29
    with pytest.raises(ValueError):
        P.StepSchedule.constant(-1.0)                    # sampling.hpp:26
    with pytest.raises(ValueError):
        P.StepSchedule.linear(0.0)                       # sampling.hpp:30
    with pytest.raises(ValueError):
        P.StepSchedule.linear(0.1, -1.0)                 # sampling.hpp:31-32
    with pytest.raises(ValueError):
        P.Ray((0, 0, 0), (1, 1, 0))                      # ray.hpp:100-101
    with pytest.raises(ValueError):
        P.Ray((0, 0, 0), (1, 0, 0), -1.0, 1.0)           # ray.hpp:102-103
    with pytest.raises(ValueError):
        P.Ray((0, 0, 0), (1, 0, 0), 2.0, 2.0)            # ray.hpp:104-105
    cam = P.Camera(width=8, height=4)
    with pytest.raises(IndexError):
        cam.pixel_ray(8, 0)                              # camera.hpp:168-169
    assert P.StepSchedule.linear(0.01, 1 / 64).step(2.0) == pytest.approx(2.0 / 64)


def test_sog_io_errors_without_gpu(P):
    """deserialize_* error paths (io.hpp:17-36,143-214) are decided before any device work."""
    g = np.load(GOLD)
    good = g["scene0_sog1"].tobytes()
    for bad, code in [(b"XXXX" + good[4:], "bad magic"), (good[:4] + b"\x02\0\0\0" + good[8:], "bad version"),
                      (good[:-5], "truncated"), (good + b"\0", "corrupt"), (good[:56] + b"\x07" + good[57:], "corrupt")]:
        with pytest.raises(P.IoError) as e:
            P.deserialize_sparse(bad)
        assert e.value.code == code
    with pytest.raises(P.IoError) as e:
        P.deserialize_dense(b"SOG0" + b"\x01\0\0\0" + b"\0" * 12)
    assert e.value.code == "truncated"


def test_sampler_create_rejects_bad_arguments(P):
    h = ctypes.c_void_p()
    assert P.lib.sogk_sampler_create(None, 1, None, ctypes.byref(h)) == P.INVALID_ARG
    assert P.lib.sogk_sample_count(None, None, 0, None, None, None, None, None) == P.INVALID_ARG


def test_ladder_seek_fuzz():
    """Closed-form ladder advance (csrc/sogk_ladder.cuh) == the reference recurrence."""
    exe = "/tmp/sogk_ladder_fuzz"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-I",
                    os.path.join(ROOT, "paper_2404_10272_b200", "csrc"), "-o", exe,
                    os.path.join(ROOT, "tests", "native", "ladder_fuzz.cpp")], check=True)
    r = subprocess.run([exe, "400000", "3"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert " 0 mismatches" in r.stdout
