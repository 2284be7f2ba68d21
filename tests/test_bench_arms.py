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
