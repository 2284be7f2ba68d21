"""Run the variant matrix (bench.hpp:514-553) on the GPU and, beside it, the unmodified
reference's run_matrix (oracle/_ref, single host thread like its default `threads = 1`), and
write both reports plus a side-by-side summary.

    python tools/matrix_compare.py --kind blobs --resolution 128 --out gpurun_out/matrix
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2404_10272_b200 import matrix as M  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="blobs")
    ap.add_argument("--resolution", type=int, default=128)
    ap.add_argument("--cascades", type=int, default=1)
    ap.add_argument("--schedule", default="constant")
    ap.add_argument("--width", type=int, default=160)
    ap.add_argument("--height", type=int, default=120)
    ap.add_argument("--out", default="gpurun_out/matrix")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    tag = f"{a.kind}_r{a.resolution}_c{a.cascades}_{a.schedule}_{a.width}x{a.height}"
    mine = M.run_matrix(M.BenchConfig(kind=a.kind, resolution=a.resolution, cascades=a.cascades,
                                      schedule=a.schedule, width=a.width, height=a.height))
    open(os.path.join(a.out, f"gpu_{tag}.json"), "w").write(M.emit_json(mine))
    open(os.path.join(a.out, f"gpu_{tag}.csv"), "w").write(M.emit_csv(mine))
    ref = None
    try:
        from oracle_bindings import RefLib

        jr, cr = RefLib().run_matrix(a.kind, resolution=a.resolution, cascades=a.cascades,
                                     sched_kind=0 if a.schedule == "constant" else 1,
                                     width=a.width, height=a.height, repetitions=5)
        open(os.path.join(a.out, f"ref_{tag}.json"), "w").write(jr)
        open(os.path.join(a.out, f"ref_{tag}.csv"), "w").write(cr)
        ref = {r["variant"]: r for r in json.loads(jr)["rows"]}
    except (OSError, FileNotFoundError) as e:
        print("reference unavailable:", e)
    lines = [f"# {tag}: GPU all_checks_passed={mine.all_checks_passed}",
             "variant,gpu_ms,ref_ms,speedup,counters_equal,gpu_psnr,gpu_conv_ms,ref_conv_ms"]
    for r in mine.rows:
        q = ref.get(r.variant) if ref else None
        if q:
            eq = (r.lookup_count, r.step_count, r.samples, r.memory_bytes) == (
                q["lookup_count"], q["step_count"], q["samples"], q["memory_bytes"])
            lines.append(f"{r.variant},{r.ms_per_frame:.4g},{q['ms_per_frame']:.4g},"
                         f"{q['ms_per_frame'] / r.ms_per_frame:.1f},{eq},{r.psnr_db:.4g},"
                         f"{r.conversion_ms:.4g},{q['conversion_ms']:.4g}")
        else:
            lines.append(f"{r.variant},{r.ms_per_frame:.4g},,,,{r.psnr_db:.4g},{r.conversion_ms:.4g},")
    txt = "\n".join(lines) + "\n"
    open(os.path.join(a.out, f"summary_{tag}.csv"), "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main()
