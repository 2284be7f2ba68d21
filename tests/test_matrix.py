"""The variant-matrix report (bench.hpp:514-605) on the GPU vs the unmodified reference.

CPU tests: our emit_csv / emit_json render the reference's own report byte for byte, and
compare_sample_sets follows bench.hpp:234-256.  GPU tests: run_matrix on the GPU gives the
reference's rows on the same config -- identical lookup / step / sample counters and memory
bytes, every check passing, PSNR equal (99 = identical images) -- timings aside.
"""
import json

import pytest

from paper_2404_10272_b200 import matrix as M


def _report_from_json(text: str) -> M.BenchReport:
    j = json.loads(text)
    sc = j["scene"]
    rep = M.BenchReport(sc["kind"], sc["seed"], sc["resolution"], sc["cascades"], sc["occupancy"],
                        all_checks_passed=j["all_checks_passed"])
    for r in j["rows"]:
        rep.rows.append(M.BenchRow(r["variant"], r["status"], r["ms_per_frame"], r["fps"],
                                   r["lookup_count"], r["step_count"], r["samples"],
                                   r["memory_bytes"], r["psnr_db"], r["conversion_ms"],
                                   list(r.get("check_messages", []))))
    return rep


@pytest.mark.parametrize("kind,cascades", [("blobs", 1), ("shell", 4)])
def test_emitters_match_reference(reflib, kind, cascades):
    jr, cr = reflib.run_matrix(kind, resolution=16, cascades=cascades, width=24, height=16)
    rep = _report_from_json(jr)
    assert M.emit_json(rep) == jr
    assert M.emit_csv(rep) == cr
    assert cr.splitlines()[0] == M.CSV_HEADER


def test_emitters_check_messages():
    rep = M.BenchReport("blobs", 1, 32, 1, 0.5)
    rep.rows.append(M.BenchRow("dense+dda+skip", "check_failed", 1.5, 666.666666, 1, 2, 3, 4, 40.123456789,
                               0.0, ["kernel twin mismatch on 3 probe rays"]))
    rep.all_checks_passed = False
    j = json.loads(M.emit_json(rep))
    assert j["schema_version"] == 1 and j["all_checks_passed"] is False
    assert j["rows"][0]["check_messages"] == ["kernel twin mismatch on 3 probe rays"]
    assert M.emit_csv(rep).splitlines()[1] == "dense+dda+skip,check_failed,1.5,666.667,1,2,3,4,40.1235,0"


def test_compare_sample_sets():
    assert M.compare_sample_sets([], []) == 0
    assert M.compare_sample_sets([1.0, 2.0], [1.0, 2.0 + 1e-12]) == 0
    assert M.compare_sample_sets([1.0, 2.0, 3.0], [1.0, 3.0]) == 1
    assert M.compare_sample_sets([1.0], [1.5, 2.0]) == 3
    assert M.nearly_equal_t(0.0, 1e-16) and not M.nearly_equal_t(0.0, 1e-14)


def test_variants():
    assert [str(v) for v in M.all_variants()] == [
        "dense+dda+branch", "dense+dda+skip", "dense+cd+branch", "dense+cd+skip",
        "sparse+hdda+branch", "sparse+hdda+skip"]
    assert str(M.REFERENCE_VARIANT) == "dense+dda+branch"


@pytest.mark.gpu
@pytest.mark.parametrize("kind,res,cascades,sched", [
    ("blobs", 32, 1, "constant"), ("shell", 32, 1, "linear"), ("sponge", 24, 1, "constant"),
    ("random", 16, 4, "constant"), ("blobs", 16, 4, "linear")])
def test_gpu_matrix_matches_reference(reflib, kind, res, cascades, sched):
    w, h = 40, 30
    jr, _ = reflib.run_matrix(kind, resolution=res, cascades=cascades,
                              sched_kind=0 if sched == "constant" else 1, width=w, height=h)
    ref = _report_from_json(jr)
    mine = M.run_matrix(M.BenchConfig(kind=kind, resolution=res, cascades=cascades, schedule=sched,
                                      width=w, height=h, repetitions=5))
    assert ref.all_checks_passed
    assert mine.all_checks_passed, [(r.variant, r.status, r.check_messages) for r in mine.rows]
    assert mine.occupancy == ref.occupancy
    assert [r.variant for r in mine.rows] == [r.variant for r in ref.rows]
    for a, b in zip(mine.rows, ref.rows):
        assert (a.lookup_count, a.step_count, a.samples, a.memory_bytes) == \
               (b.lookup_count, b.step_count, b.samples, b.memory_bytes), a.variant
        assert a.psnr_db == b.psnr_db, a.variant
        assert a.ms_per_frame > 0 and a.fps > 0
        assert (a.conversion_ms > 0) == (b.conversion_ms > 0)
    text = M.emit_json(mine)
    assert json.loads(text)["schema_version"] == 1
    assert M.emit_csv(mine).splitlines()[0] == M.CSV_HEADER
