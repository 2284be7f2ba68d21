"""The reference bench's variant matrix (bench.hpp:514-553) on the GPU, in its report schema.

`run_matrix(cfg)` renders one frame per variant of the reference's matrix
(`all_variants`, bench.hpp:45-54: dense+dda, dense+cd, sparse+hdda, each with +branch and +skip)
with the GPU sampler and compositor and fills the reference's `BenchRow` fields
(bench.hpp:259-271): median ms per frame over >= 5 frames, fps, the FrameResult counters,
`variant_memory_bytes` (bench.hpp:463-476), PSNR against the reference variant's frame
(dense+dda+branch) and the grid conversion time (median of 10 builds).  The alongside checks
of `run_row_checks` (bench.hpp:483-512) run on the same probe pixels: the kernel twin must give
identical sample buffers and the sample set must match the reference analyzer's within
`compare_sample_sets`' tolerance.  `emit_csv` / `emit_json` write the reference's formats
(bench.hpp:555-605: fixed CSV columns, schema_version 1).

    python -m paper_2404_10272_b200.matrix --kind shell --seed 1 --resolution 128 \\
        --width 160 --height 120 --out-json report.json --out-csv report.csv
"""
from __future__ import annotations

import argparse
import json
import statistics
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import (Analyzer, Camera, GridTransform, KernelKind, Sampler, StepSchedule, analytic_scene,
               build_dense_cascade, build_distance, build_sparse, generate_scene, psnr, render_frame,
               DenseGrid)

CSV_HEADER = ("variant,status,ms_per_frame,fps,lookup_count,step_count,samples,memory_bytes,psnr_db,"
              "conversion_ms")  # kCsvHeader, bench.hpp:559-561
DEFAULT_LINEAR_GROWTH = 1.0 / 256.0  # kDefaultLinearGrowth (sampling.hpp:12)


@dataclass
class VariantId:  # bench.hpp:30-37
    grid: str       # "dense" | "sparse"
    analyzer: str   # "dda" | "hdda" | "cd"
    kernel: str     # "branch" | "skip"

    def __str__(self) -> str:
        return f"{self.grid}+{self.analyzer}+{self.kernel}"


def all_variants() -> List[VariantId]:  # bench.hpp:45-54
    return [VariantId("dense", "dda", "branch"), VariantId("dense", "dda", "skip"),
            VariantId("dense", "cd", "branch"), VariantId("dense", "cd", "skip"),
            VariantId("sparse", "hdda", "branch"), VariantId("sparse", "hdda", "skip")]


REFERENCE_VARIANT = VariantId("dense", "dda", "branch")  # kReferenceVariant, bench.hpp:64


@dataclass
class BenchConfig:  # bench.hpp:71-96 (the fields the matrix uses)
    kind: str = "blobs"
    seed: int = 1
    fraction: float = 0.05
    count: int = 12
    threshold: float = 0.01
    resolution: int = 128
    cascades: int = 1
    schedule: str = "constant"
    dt0: float = 0.0  # 0 = half the finest voxel
    growth: float = DEFAULT_LINEAR_GROWTH
    width: int = 160
    height: int = 120
    repetitions: int = 5
    variants: List[VariantId] = field(default_factory=all_variants)


@dataclass
class BenchRow:  # bench.hpp:259-271
    variant: str
    status: str = "ok"
    ms_per_frame: float = 0.0
    fps: float = 0.0
    lookup_count: int = 0
    step_count: int = 0
    samples: int = 0
    memory_bytes: int = 0
    psnr_db: float = 0.0
    conversion_ms: float = 0.0
    check_messages: List[str] = field(default_factory=list)


@dataclass
class BenchReport:  # bench.hpp:273-281
    scene: str
    seed: int
    resolution: int
    cascades: int
    occupancy: float
    rows: List[BenchRow] = field(default_factory=list)
    all_checks_passed: bool = True


def nearly_equal_t(a: float, b: float, rel: float = 1e-9) -> bool:  # bench.hpp:197-199
    return abs(a - b) <= rel * max(abs(a), abs(b)) + 1e-15


def compare_sample_sets(a, b, rel: float = 1e-9) -> int:
    """`differing` of compare_sample_sets (bench.hpp:234-256): samples present on one side only."""
    i = j = diff = 0
    while i < len(a) and j < len(b):
        if nearly_equal_t(a[i], b[j], rel):
            i += 1
            j += 1
        elif a[i] < b[j]:
            diff += 1
            i += 1
        else:
            diff += 1
            j += 1
    return diff + (len(a) - i) + (len(b) - j)


def _time_ms(fn, reps: int) -> float:
    import torch

    times = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    return statistics.median(times)


class _Assets:
    """build_assets (bench.hpp:306-376) with the grids in HBM."""

    def __init__(self, cfg: BenchConfig):
        base = GridTransform.cube(cfg.resolution, (-1.0, -1.0, -1.0), 2.0)
        bits, self.occupancy = generate_scene(cfg.kind, base, seed=cfg.seed, fraction=cfg.fraction,
                                              count=cfg.count, threshold=cfg.threshold)
        self.scene = analytic_scene(cfg.kind, base, seed=cfg.seed, count=cfg.count)
        if cfg.cascades == 1:
            levels = [(base, bits)]
        elif cfg.kind == "random":  # coarser levels reuse the level-0 bits (bench.hpp:334-343)
            levels = [(GridTransform(base.resolution, (-(2.0 ** b),) * 3, base.voxel_size * 2 ** b), bits)
                      for b in range(cfg.cascades)]
        else:
            levels = build_dense_cascade(cfg.kind, base, cfg.cascades, seed=cfg.seed,
                                         fraction=cfg.fraction, count=cfg.count,
                                         threshold=cfg.threshold)
        self.dense = [DenseGrid(t, b) for t, b in levels]
        self.sparse_ms = _time_ms(lambda: [build_sparse(d) for d in self.dense], 10)
        self.sparse = [build_sparse(d) for d in self.dense]
        self.distance_ms = _time_ms(lambda: [build_distance(d) for d in self.dense], 10)
        self.distance = [build_distance(d) for d in self.dense]
        self.camera = Camera((1.9, 1.4, 2.3), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 42.0, cfg.width, cfg.height)
        dt0 = cfg.dt0 if cfg.dt0 > 0.0 else 0.5 * base.voxel_size
        self.schedule = (StepSchedule.constant(dt0) if cfg.schedule == "constant"
                         else StepSchedule.linear(dt0, cfg.growth))
        self.cascade = cfg.cascades > 1

    def sampler(self, v: VariantId) -> Sampler:  # make_sampler (bench.hpp:382-413)
        an = {"dda": Analyzer.dda, "hdda": Analyzer.hdda, "cd": Analyzer.cd}[v.analyzer]
        grids = {"dda": self.dense, "hdda": self.sparse, "cd": self.distance}[v.analyzer]
        k = KernelKind.branch if v.kernel == "branch" else KernelKind.skip
        return Sampler(grids, an, k, self.schedule, cascade=self.cascade)

    def memory_bytes(self, v: VariantId) -> int:  # variant_memory_bytes (bench.hpp:463-476)
        if v.grid == "sparse":
            return sum(g.memory_bytes() for g in self.sparse)
        total = sum(g.memory_bytes() for g in self.dense)
        if v.analyzer == "cd":
            total += sum(g.transform().voxel_count() * 4 for g in self.dense)
        return total


def _row_checks(a: _Assets, v: VariantId, row: BenchRow):
    """run_row_checks (bench.hpp:483-512) on the probe pixels every total/512-th."""
    cam = a.camera
    total = cam.width * cam.height
    stride = max(1, total // 512)
    rays = cam.rays()[::stride]
    twin = VariantId(v.grid, v.analyzer, "skip" if v.kernel == "branch" else "branch")

    def buffers(var):
        out = a.sampler(var).sample_host(rays)
        pi = out.packed_info
        return [out.t_starts[pi[r, 0]:pi[r, 0] + pi[r, 1]] for r in range(rays.shape[0])]

    mine, tw, ref = buffers(v), buffers(twin), buffers(REFERENCE_VARIANT)
    kernel_mismatches = sum(not np.array_equal(x, y) for x, y in zip(mine, tw))
    analyzer_mismatches = sum(compare_sample_sets(x, y) > 0 for x, y in zip(mine, ref))
    if kernel_mismatches:
        row.status = "check_failed"
        row.check_messages.append(f"kernel twin mismatch on {kernel_mismatches} probe rays")
    if analyzer_mismatches:
        row.status = "check_failed"
        row.check_messages.append(f"sample set deviates from reference on {analyzer_mismatches} probe rays")


def run_matrix(cfg: BenchConfig) -> BenchReport:  # bench.hpp:514-553
    a = _Assets(cfg)
    report = BenchReport(cfg.kind, cfg.seed, cfg.resolution, cfg.cascades, a.occupancy)
    reference_image = render_frame(a.sampler(REFERENCE_VARIANT), a.scene, a.camera).image
    for v in cfg.variants:
        row = BenchRow(str(v))
        try:
            s = a.sampler(v)
            counted = render_frame(s, a.scene, a.camera)
            row.lookup_count, row.step_count, row.samples = counted.lookups, counted.steps, counted.samples
            row.memory_bytes = a.memory_bytes(v)
            row.ms_per_frame = _time_ms(lambda: render_frame(s, a.scene, a.camera), max(5, cfg.repetitions))
            row.fps = 1000.0 / row.ms_per_frame if row.ms_per_frame > 0 else 0.0
            row.psnr_db = psnr(counted.image, reference_image)
            row.conversion_ms = (a.sparse_ms if v.grid == "sparse" else a.distance_ms if v.analyzer == "cd"
                                 else 0.0)
            _row_checks(a, v, row)
        except Exception as e:  # noqa: BLE001  (a failed row is reported, like the reference)
            row.status = f"failed: {e}"
        if row.status != "ok":
            report.all_checks_passed = False
        report.rows.append(row)
    return report


def emit_csv(report: BenchReport) -> str:  # bench.hpp:563-578 (%.6g numbers)
    lines = [CSV_HEADER]
    for r in report.rows:
        lines.append(",".join([r.variant, r.status, f"{r.ms_per_frame:.6g}", f"{r.fps:.6g}",
                               str(r.lookup_count), str(r.step_count), str(r.samples),
                               str(r.memory_bytes), f"{r.psnr_db:.6g}", f"{r.conversion_ms:.6g}"]))
    return "\n".join(lines) + "\n"


def emit_json(report: BenchReport) -> str:  # bench.hpp:580-605, schema_version 1
    rows = []
    for r in report.rows:
        d = {"variant": r.variant, "status": r.status, "ms_per_frame": r.ms_per_frame, "fps": r.fps,
             "lookup_count": r.lookup_count, "step_count": r.step_count, "samples": r.samples,
             "memory_bytes": r.memory_bytes, "psnr_db": r.psnr_db, "conversion_ms": r.conversion_ms}
        if r.check_messages:
            d["check_messages"] = r.check_messages
        rows.append(d)
    j = {"schema_version": 1,
         "scene": {"kind": report.scene, "seed": report.seed, "resolution": report.resolution,
                   "cascades": report.cascades, "occupancy": report.occupancy},
         "all_checks_passed": report.all_checks_passed, "rows": rows}
    return json.dumps(j, indent=2, sort_keys=True)  # nlohmann::json objects are key-ordered


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--kind", default="blobs", choices=["blobs", "shell", "sponge", "random"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--fraction", type=float, default=0.05)
    ap.add_argument("--resolution", type=int, default=128)
    ap.add_argument("--cascades", type=int, default=1, choices=[1, 4])
    ap.add_argument("--schedule", default="constant", choices=["constant", "linear"])
    ap.add_argument("--width", type=int, default=160)
    ap.add_argument("--height", type=int, default=120)
    ap.add_argument("--repetitions", type=int, default=5)
    ap.add_argument("--out-json", default="")
    ap.add_argument("--out-csv", default="")
    args = ap.parse_args(argv)
    cfg = BenchConfig(kind=args.kind, seed=args.seed, fraction=args.fraction, resolution=args.resolution,
                      cascades=args.cascades, schedule=args.schedule, width=args.width, height=args.height,
                      repetitions=args.repetitions)
    rep = run_matrix(cfg)
    if args.out_json:
        open(args.out_json, "w").write(emit_json(rep))
    if args.out_csv:
        open(args.out_csv, "w").write(emit_csv(rep))
    print(emit_csv(rep), end="")
    return 0 if rep.all_checks_passed else 1


if __name__ == "__main__":
    raise SystemExit(main())
