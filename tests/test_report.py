"""Result files vs the reference's own output directory (tests/golden/report_golden.json, made by
tests/golden/make_report_golden.py from rigaeig's cli.run_experiment).

CPU tests pin the formats: tables re-rendered from the parsed golden values must reproduce the reference's
text byte for byte, and the manifest its schema.  The GPU test solves the same level sweep on the device and
compares numerically."""
import hashlib
import json
import os
from dataclasses import dataclass

import numpy as np
import pytest

from paper_2009_08167_b200.report import (ERRORS_COLUMNS, SPECTRUM_COLUMNS, SWEEP_COLUMNS, artifact_names,
                                          cost_report, errors_csv, report_json, spectrum_csv, sweep_csv,
                                          sweep_row, write_artifacts)
from paper_2009_08167_b200.sparsela import CostCounters

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "report_golden.json")))
D, NE, P_, N_IGA = 1, 16, 3, 17


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


def _counters(fact, fb, mv, calls, nsh=None, nit=14):
    c = CostCounters()
    c.fact.flops, c.fb.flops, c.matvec.flops = fact, fb, mv
    c.fact.calls, c.fb.calls, c.matvec.calls = calls
    c.fact.seconds, c.fb.seconds, c.matvec.seconds = 0.5, 0.25, 0.125
    c.nsh, c.nit = calls[0] if nsh is None else nsh, nit
    return c


def _golden_files(level):
    """The level's three files re-rendered from the golden values."""
    names = artifact_names(D, NE, P_, level)
    _, srows = _csv(GOLD["files"][names["spectrum"]])
    spec = spectrum_csv([float(r[1]) for r in srows], [float(r[2]) for r in srows], [int(r[3]) for r in srows])
    _, erows = _csv(GOLD["files"][names["errors"]])
    errs = errors_csv([_Rec(int(r[0]) - 1, float(r[2]), float(r[3]), float(r[4]), r[5] == "1") for r in erows],
                      N_IGA)
    g = json.loads(GOLD["files"][names["report"]])
    c = _counters(g["flops"]["fact"], g["flops"]["fb"], g["flops"]["matvec"],
                  (g["counters"]["Nfa"], g["counters"]["Nfb"], g["counters"]["Nmv"]), g["counters"]["Nsh"],
                  g["counters"]["Nit"])
    rep = cost_report(g["config"], c)
    rep["time_s"] = g["time_s"]  # wall seconds are run-specific
    return names, spec, errs, report_json(rep), c


def test_tables_reproduce_reference_text():
    for level in (0, 1):
        names, spec, errs, rep, _ = _golden_files(level)
        assert spec == GOLD["files"][names["spectrum"]]
        assert errs == GOLD["files"][names["errors"]]
        assert rep == GOLD["files"][names["report"]]
    assert ",".join(SPECTRUM_COLUMNS) == GOLD["files"][names["spectrum"]].split("\n")[0]
    assert ",".join(ERRORS_COLUMNS) == GOLD["files"][names["errors"]].split("\n")[0]


def test_error_rows_print_nan():
    assert errors_csv([_Rec(0, 1.5e-3, float("nan"), float("nan"), False)], 4).split("\n")[1] == \
        "1,0.25,1.500000000000e-03,nan,nan,0"


def test_sweep_table_reproduces_reference_text():
    sweep_name = artifact_names(D, NE, P_)["sweep"]
    hdr, rows = _csv(GOLD["files"][sweep_name])
    assert hdr == ",".join(SWEEP_COLUMNS)
    out = []
    for r in rows:
        v = dict(zip(SWEEP_COLUMNS, (int(x) for x in r)))
        c = _counters(v["fact_flops"], v["fb_flops"], v["matvec_flops"], (v["Nfa"], v["Nfb"], v["Nmv"]), v["Nsh"],
                      v["Nit"])
        out.append(sweep_row(v["level"], v["blocksize"], v["N"], v["nnz_K"], v["fill_nnz"], c))
    assert sweep_csv(out) == GOLD["files"][sweep_name]


def test_manifest_matches_reference_schema(tmp_path):
    files = []
    for level in (0, 1):
        names, spec, errs, rep, _ = _golden_files(level)
        files += [(names["spectrum"], spec), (names["errors"], errs), (names["report"], rep)]
    sweep_name = artifact_names(D, NE, P_)["sweep"]
    files.append((sweep_name, GOLD["files"][sweep_name]))
    mpath = write_artifacts(tmp_path, files, GOLD["config"], [(0, "ok"), (1, "ok")], seed=0)
    man = json.loads(mpath.read_text())
    assert sorted(man) == GOLD["manifest_keys"]
    assert [f["path"] for f in man["files"]] == GOLD["manifest_files"]
    assert man["config_sha256"] == GOLD["config_sha256"]
    assert not man["partial"]
    for f in man["files"]:
        p = tmp_path / f["path"]
        assert p.read_text() == GOLD["files"][f["path"]]
        assert f["sha256"] == hashlib.sha256(p.read_bytes()).hexdigest() and f["bytes"] == p.stat().st_size
    part = json.loads(write_artifacts(tmp_path / "b", [], GOLD["config"], [(0, "ok"), (1, "count-mismatch")],
                                      0).read_text())
    assert part["partial"] and {"level": 1, "status": "count-mismatch"} in part["points"]


def test_cost_report_schema():
    g = json.loads(GOLD["files"][artifact_names(D, NE, P_, 0)["report"]])
    rep = cost_report(g["config"], _counters(1, 2, 3, (4, 5, 6)))
    assert set(rep) == set(g) and set(rep["time_s"]) == set(g["time_s"])
    assert rep["time_s"]["total"] == pytest.approx(0.875)


@pytest.mark.gpu
def test_device_sweep_matches_reference_files(tmp_path):
    """The reference's level sweep (1D, ne=16, p=3, levels 0 and 1, 10 eigenpairs) solved on the device,
    written through the writers, compared with the reference's files."""
    import paper_2009_08167_b200 as P

    cfg = GOLD["config"]
    files, sweep, points = [], [], []
    for level in cfg["levels"]:
        system = P.build_system(cfg["d"], cfg["ne"], cfg["p"], level)
        res = P.solve_spectrum(system, count=cfg["nev"], seed=cfg["seed"] + level, m=cfg["lanczos_m"],
                               keep=cfg["keep"], tol=cfg["tol"])
        records = P.error_table(res.eigenvalues, res.vectors, system)
        names = artifact_names(cfg["d"], cfg["ne"], cfg["p"], level)
        conf = {"d": cfg["d"], "ne": cfg["ne"], "p": cfg["p"], "level": level, "N": system.dof_count,
                "N0": cfg["nev"]}
        files += [(names["spectrum"], spectrum_csv(res.eigenvalues, res.residuals, res.slice_ids)),
                  (names["errors"], errors_csv(records, N_IGA)),
                  (names["report"], report_json(cost_report(conf, res.counters)))]
        fill = P.factor_ldl(system.K, ordering=P.separator_ordering(system)).fill_nnz
        sweep.append(sweep_row(level, 2 ** (cfg["ne"].bit_length() - 1 - level), system.dof_count, system.K.nnz,
                               fill, res.counters))
        points.append((level, "ok"))
    files.append((artifact_names(cfg["d"], cfg["ne"], cfg["p"])["sweep"], sweep_csv(sweep)))
    write_artifacts(tmp_path, files, cfg, points, cfg["seed"])
    assert sorted(name for name, _ in files) == sorted(GOLD["files"])
    for level in cfg["levels"]:
        names = artifact_names(cfg["d"], cfg["ne"], cfg["p"], level)
        h, got = _csv((tmp_path / names["spectrum"]).read_text())
        _, ref = _csv(GOLD["files"][names["spectrum"]])
        assert len(got) == len(ref) and [r[0] for r in got] == [r[0] for r in ref]
        np.testing.assert_allclose([float(r[1]) for r in got], [float(r[1]) for r in ref], rtol=1e-10)
        assert max(float(r[2]) for r in got) < 1e-8
        _, got = _csv((tmp_path / names["errors"]).read_text())
        _, ref = _csv(GOLD["files"][names["errors"]])
        assert [r[:2] + r[5:] for r in got] == [r[:2] + r[5:] for r in ref]
        for col in (2, 3, 4):
            np.testing.assert_allclose([float(r[col]) for r in got], [float(r[col]) for r in ref], rtol=1e-4,
                                       atol=1e-11)
        rep = json.loads((tmp_path / names["report"]).read_text())
        assert rep["config"] == json.loads(GOLD["files"][names["report"]])["config"]
    _, got = _csv((tmp_path / artifact_names(cfg["d"], cfg["ne"], cfg["p"])["sweep"]).read_text())
    _, ref = _csv(GOLD["files"][artifact_names(cfg["d"], cfg["ne"], cfg["p"])["sweep"]])
    for g, r in zip(got, ref):
        assert g[:5] == r[:5]  # level, blocksize, N, nnz_K, fill_nnz
