"""Experiment artifacts and cost reports vs the reference's own output directory (tests/golden/report_golden.json,
made by tests/golden/make_report_golden.py from rigaeig's cli.run_experiment).

CPU tests pin the formats (rows re-rendered from the parsed golden values must reproduce the reference's text
byte for byte) and the cost model; the GPU test runs the same sweep through the device solve."""
import json
import math
import os
from dataclasses import dataclass

import numpy as np
import pytest

from paper_2009_08167_b200.costmodel import (RunReport, TimeModel, improvement_report, predict_factor_flops,
                                             predict_fb_flops, predict_time, time_exponents)
from paper_2009_08167_b200.report import (ERRORS_HEADER, SPECTRUM_HEADER, ConfigError, ExperimentConfig,
                                          PointResult, _levels, error_rows, load_config, spectrum_rows,
                                          write_bundle)
from paper_2009_08167_b200.sparsela import CostCounters

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "report_golden.json")))
BASE = "d1_ne16_p3"


def _cfg(out):
    c = GOLD["config"]
    return ExperimentConfig(d=c["d"], ne=c["ne"], p=c["p"], levels=c["levels"], nev=c["nev"], out=str(out),
                            seed=c["seed"], figures=False)


def _csv(text):
    lines = text.strip().split("\n")
    return lines[0], [ln.split(",") for ln in lines[1:]]


@dataclass
class _Rec:
    position: int
    ev: float
    efl: float
    efe: float
    diagonal: bool


def _golden_point(level):
    tag = f"{BASE}_l{level}"
    _, srows = _csv(GOLD["files"][f"spectrum_{tag}.csv"])
    lam = [float(r[1]) for r in srows]
    res = [float(r[2]) for r in srows]
    sid = [int(r[3]) for r in srows]
    _, erows = _csv(GOLD["files"][f"errors_{tag}.csv"])
    recs = [_Rec(int(r[0]) - 1, float(r[2]), float(r[3]), float(r[4]), r[5] == "1") for r in erows]
    report = json.loads(GOLD["files"][f"report_{tag}.json"])
    hdr, wrows = _csv(GOLD["files"][f"sweep_{BASE}.csv"])
    cols = hdr.split(",")
    sweep = [dict(zip(cols, (int(v) for v in r))) for r in wrows if int(r[0]) == level][0]
    return PointResult(level, "ok", spectrum_rows(lam, res, sid), error_rows(recs, 17), report, sweep)


def test_rows_reproduce_reference_text():
    for level in (0, 1):
        tag = f"{BASE}_l{level}"
        pt = _golden_point(level)
        assert "\n".join([SPECTRUM_HEADER] + pt.spectrum_rows) + "\n" == GOLD["files"][f"spectrum_{tag}.csv"]
        assert "\n".join([ERRORS_HEADER] + pt.error_rows) + "\n" == GOLD["files"][f"errors_{tag}.csv"]


def test_error_rows_print_nan():
    rows = error_rows([_Rec(0, 1.5e-3, float("nan"), float("nan"), False)], 4)
    assert rows == ["1,0.25,1.500000000000e-03,nan,nan,0"]


def test_bundle_matches_reference_directory(tmp_path):
    cfg = _cfg(tmp_path)
    bundle = write_bundle(cfg, [_golden_point(0), _golden_point(1)])
    names = sorted(f.name for f in bundle.files)
    assert names == sorted(GOLD["files"])
    for f in bundle.files:
        assert f.read_text() == GOLD["files"][f.name], f.name
    man = json.loads(bundle.manifest_path.read_text())
    assert sorted(man) == GOLD["manifest_keys"]
    assert [f["path"] for f in man["files"]] == GOLD["manifest_files"]
    assert man["config_sha256"] == GOLD["config_sha256"]
    assert not man["partial"] and bundle.failed_points == []
    import hashlib
    for f in man["files"]:
        p = tmp_path / f["path"]
        assert f["sha256"] == hashlib.sha256(p.read_bytes()).hexdigest() and f["bytes"] == p.stat().st_size


def test_failed_point_marks_manifest_partial(tmp_path):
    bundle = write_bundle(_cfg(tmp_path), [_golden_point(0), PointResult(1, "count-mismatch: x")])
    man = json.loads(bundle.manifest_path.read_text())
    assert man["partial"] and bundle.failed_points == [1]
    assert {"level": 1, "status": "count-mismatch: x"} in man["points"]


def test_config_validation_and_loading(tmp_path):
    ExperimentConfig(nev=5).validate()
    for bad in (dict(d=4, nev=5), dict(ne=12, nev=5), dict(p=0, nev=5), dict(levels=[], nev=5),
                dict(levels=[9], nev=5), dict(), dict(nev=5, interval=(0, 1)), dict(nev="all"), dict(nev=0),
                dict(interval=(2.0, 1.0)), dict(nev=5, lanczos_m=3), dict(nev=5, keep=59),
                dict(nev=5, workers=0)):
        with pytest.raises(ConfigError):
            ExperimentConfig(**bad).validate()
    assert ExperimentConfig(ne=16, p=3, nev="niga").resolved_nev(1) == 17
    assert ExperimentConfig(ne=16, p=3, nev=100).resolved_nev(0) == 17
    assert _levels("0-2,5") == [0, 1, 2, 5]
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"d": 2, "ne": 8, "nev": "12", "interval": None}))
    cfg = load_config(str(p), p=2)
    assert (cfg.d, cfg.ne, cfg.p, cfg.nev) == (2, 8, 2, 12)
    p.write_text(json.dumps({"dee": 2}))
    with pytest.raises(ConfigError):
        load_config(str(p))
    p.write_text("{")
    with pytest.raises(ConfigError):
        load_config(str(p))


def _counters(fact, fb, mv, calls):
    c = CostCounters()
    c.fact.flops, c.fb.flops, c.matvec.flops = fact, fb, mv
    c.fact.calls, c.fb.calls, c.matvec.calls = calls
    c.fact.seconds, c.fb.seconds, c.matvec.seconds = 0.5, 0.25, 0.125
    c.nsh, c.nit = calls[0], 14
    return c


def test_run_report_schema_matches_reference():
    g = json.loads(GOLD["files"][f"report_{BASE}_l0.json"])
    c = _counters(g["flops"]["fact"], g["flops"]["fb"], g["flops"]["matvec"],
                  (g["counters"]["Nfa"], g["counters"]["Nfb"], g["counters"]["Nmv"]))
    rep = RunReport.from_counters(g["config"], c).to_json_dict()
    assert set(rep) == set(g) and set(rep["time_s"]) == set(g["time_s"])
    assert rep["counters"] == g["counters"] and rep["flops"] == g["flops"] and rep["config"] == g["config"]
    assert rep["time_s"]["total"] == pytest.approx(0.875)


def test_cost_model_predictions():
    np.testing.assert_allclose(predict_factor_flops(4 * 4096, 3, 0, 2) / predict_factor_flops(4096, 3, 0, 2), 8.0)
    np.testing.assert_allclose(predict_fb_flops(4 * 4096, 3, 0, 2) / predict_fb_flops(4096, 3, 0, 2), 4.0)
    # partitioning: 2^(d level) blocks plus the separator skeleton
    N = 4096.0
    assert predict_factor_flops(N, 3, 2, 2) == pytest.approx(16 * (N / 16) ** 1.5 * 27 + N ** 1.5)
    assert predict_factor_flops(N, 3, 2, 2) < predict_factor_flops(N, 3, 0, 2)
    assert time_exponents("fact", "iga", 3) == (2.0, 3.0)
    assert time_exponents("fb", "riga", 2) == (1.0, 1.0)
    assert time_exponents("matvec", "iga", 3) == (1.0, 3.0)
    with pytest.raises(ValueError):
        time_exponents("lu", "iga", 2)
    with pytest.raises(ValueError):
        time_exponents("fact", "fem", 2)
    m = TimeModel.calibrate("fact", "iga", 2, 1000, 3, 2.0)
    assert m.predict(1000, 3) == pytest.approx(2.0)
    assert predict_time("fact", "iga", 2, (1000, 3, 2.0), 4000, 3) == pytest.approx(2.0 * 4 ** 1.5)
    with pytest.raises(ValueError):
        m.predict(64 * 1000 + 1, 3)
    with pytest.raises(ValueError):
        TimeModel.calibrate("fact", "iga", 2, 1000, 3, 0.0)


def test_improvement_report():
    cfg = {"d": 1, "ne": 16, "p": 3, "N0": 10}
    a = RunReport.from_counters(cfg, _counters(100, 50, 10, (5, 50, 100)))
    same = improvement_report(a, a)
    assert all(v == pytest.approx(1.0) for v in same["flops"].values()) and not same["matvec_degraded"]
    b = RunReport.from_counters(cfg, _counters(400, 100, 5, (5, 50, 100)))  # IGA costlier except mat-vec
    rep = improvement_report(a, b)
    assert rep["flops"]["fact"] == pytest.approx(4.0) and rep["flops"]["total"] == pytest.approx(505 / 160)
    assert rep["matvec_degraded"] and a.ratios_vs_baseline["flops"] == rep["flops"]
    other = RunReport.from_counters(dict(cfg, p=2), _counters(1, 1, 1, (1, 1, 1)))
    with pytest.raises(ValueError):
        improvement_report(other, a)
    z = RunReport.from_counters(cfg, _counters(0, 1, 1, (1, 1, 1)))
    assert math.isinf(improvement_report(z, a)["flops"]["fact"])


@pytest.mark.gpu
def test_run_experiment_on_device_matches_reference(tmp_path):
    from paper_2009_08167_b200.report import run_experiment

    bundle = run_experiment(_cfg(tmp_path))
    assert sorted(f.name for f in bundle.files) == sorted(GOLD["files"]) and not bundle.failed_points
    for level in (0, 1):
        tag = f"{BASE}_l{level}"
        h, got = _csv((tmp_path / f"spectrum_{tag}.csv").read_text())
        _, ref = _csv(GOLD["files"][f"spectrum_{tag}.csv"])
        assert h == SPECTRUM_HEADER and len(got) == len(ref)
        np.testing.assert_allclose([float(r[1]) for r in got], [float(r[1]) for r in ref], rtol=1e-10)
        assert max(float(r[2]) for r in got) < 1e-8
        assert [r[0] for r in got] == [r[0] for r in ref]
        h, got = _csv((tmp_path / f"errors_{tag}.csv").read_text())
        _, ref = _csv(GOLD["files"][f"errors_{tag}.csv"])
        assert h == ERRORS_HEADER and [r[:2] + r[5:] for r in got] == [r[:2] + r[5:] for r in ref]
        for col, atol in ((2, 1e-11), (3, 1e-11), (4, 1e-11)):
            np.testing.assert_allclose([float(r[col]) for r in got], [float(r[col]) for r in ref], rtol=1e-4,
                                       atol=atol)
        rep = json.loads((tmp_path / f"report_{tag}.json").read_text())
        gref = json.loads(GOLD["files"][f"report_{tag}.json"])
        assert rep["config"] == gref["config"]
        assert rep["counters"]["Nfa"] >= rep["counters"]["Nsh"] >= 1
    hdr, got = _csv((tmp_path / f"sweep_{BASE}.csv").read_text())
    ghdr, ref = _csv(GOLD["files"][f"sweep_{BASE}.csv"])
    assert hdr == ghdr
    for g, r in zip(got, ref):
        assert g[:5] == r[:5]  # level, blocksize, N, nnz_K, fill_nnz
