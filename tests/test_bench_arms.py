"""bench.py's reference arm: the unmodified reference sampler with inputs from the
reference's own generators; it must never load the product library (libsogk.so) and must
print the same `config` as the GPU arm (the driver's same_config check)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_never_loads_the_product_library():
    code = (
        "import sys, runpy, json, io, contextlib\n"
        "sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0','--cpu-stride','512']\n"
        "buf = io.StringIO()\n"
        "with contextlib.redirect_stdout(buf):\n"
        "    runpy.run_path('bench.py', run_name='__main__')\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'line': buf.getvalue().strip().splitlines()[-1], 'sogk': 'libsogk' in maps,\n"
        "                  'pkg': any(m.startswith('paper_2404_10272_b200') for m in sys.modules),\n"
        "                  'ref': 'libsogref' in maps}))\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    line = json.loads(out["line"])
    if "unavailable" in line:  # oracle/_ref not built on this host
        return
    assert not out["sogk"] and not out["pkg"], "the reference arm loaded the product library"
    assert out["ref"]
    sys.path.insert(0, ROOT)
    import bench

    assert line["config"] == bench.workload_config("cfg2", 1, 2)
    assert line["impl"] == "reference" and line["value"] > 0


def test_workload_shards_cover_the_step_once():
    """SURVEY §8e partitioning as bench.py does it: cfg1/3/4 contiguous ceil(N/G) ray ranges that
    tile the step's rays exactly once for every world size (global ray_indices = range start);
    cfg2 one distinct orbit view per rank per object (weak scaling)."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2404_10272_b200 as P

    wl = bench.Workload("cfg1", bench.ProductGen(P))
    n = wl.frame_rays()
    for world in (1, 2, 3, 8):
        specs = [wl.shard(0, 0, r, world) for r in range(world)]
        assert specs[0]["first"] == 0
        for a, b in zip(specs, specs[1:]):
            assert a["first"] + a["count"] == b["first"]
        assert specs[-1]["first"] + specs[-1]["count"] == n
        assert bench.workload_config("cfg1", world, 2)["rays_per_step"] == n  # strong scaling
    wl2 = bench.Workload("cfg2", bench.ProductGen(P))
    for world in (1, 2, 8):
        views = {(o, wl2.shard(3, o, r, world)["pos"]) for o in range(8) for r in range(world)}
        assert len(views) == 8 * world
        assert bench.workload_config("cfg2", world, 2)["rays_per_step"] == 8 * 800 * 800 * world
    assert bench.scaling_of("cfg2") == "weak" and bench.scaling_of("cfg4") == "strong"


def test_host_expand_link_bytes(monkeypatch):
    sys.path.insert(0, ROOT)
    import bench

    for mode, b in (("t", 12), ("all", 8), ("ri", 16), ("0", 20)):
        monkeypatch.setenv("SOGK_HOST_EXPAND", mode)
        assert bench.host_expand_link_bytes() == b
    monkeypatch.delenv("SOGK_HOST_EXPAND")
    assert bench.host_expand_link_bytes() == 12
