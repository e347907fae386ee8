"""Benchmark rows in the reference's report schema.

report.py writes what report_to_csv (src/report.cpp:180-198) writes; the pin
is the reference's own code: tests/cpp/ref_report reads our CSV with
read_report_csv and writes it back with report_to_csv, and the bytes must not
change.
"""
from __future__ import annotations

import math
import os
import subprocess

import pytest

import paper_2510_05254_b200 as ndgx
from paper_2510_05254_b200 import report as rp

REF_REPORT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "ref_report")


def _ref_roundtrip(tmp_path, text):
    if not os.path.exists(REF_REPORT):
        pytest.skip("tests/cpp/_build/ref_report not built (needs /root/reference at build time)")
    p = tmp_path / "ours.csv"
    p.write_text(text)
    return subprocess.run([REF_REPORT, str(p)], check=True, capture_output=True, text=True).stdout


def _rows():
    a = rp.BenchRow(experiment="timing", equation="euler", dim=2, order=8, rk="rk4", nx=1250, ny=1250, cfl=0.4,
                    workers=1, dof=300_000_000, device="B200 (sm_100a)", steps=5, dt_min=1.0 / 3.0,
                    dt_max=2.5e-7, wall_seconds=0.0142, note="fast, contracted")
    a.time_per_dof = a.wall_seconds / a.dof
    b = rp.BenchRow(experiment="scale", row_type="run", status="failed", equation="advection", dim=3, order=4,
                    rk="rk6", nx=96, ny=96, nz=48, nk=7, seed=2**63 + 5, workers=8, dof=10**12,
                    note='say "hi", then stop', speedup=7.25, efficiency=0.90625)
    c = rp.BenchRow(experiment="x", row_type="warning", status="skipped", note="", steps=0, l2_error=1e-300,
                    slope=-4.0000000000000009, fit_c=float("inf"), energy_per_dof=-0.0)
    return [a, b, c]


def test_csv_escape_and_double_format():
    assert rp.csv_escape("plain") == "plain"
    assert rp.csv_escape('a,"b"') == '"a,""b"""'
    # quoted like csv_escape; the reference's line-based reader cannot read it back
    assert rp.csv_escape("a\nb") == '"a\nb"'
    assert rp.fmt_double(float("nan")) == "" and rp.fmt_double(0.1) == "0.10000000000000001"
    row = rp.BenchRow()
    cells = rp.report_to_csv(rp.BenchReport(rows=[row])).splitlines()[3].split(",")
    assert len(cells) == len(rp.COLUMNS) == 33
    assert cells[rp.COLUMNS.index("steps")] == "" and cells[rp.COLUMNS.index("row_type")] == "run"


def test_csv_is_byte_identical_through_the_reference_reader_and_writer(tmp_path):
    rep = rp.BenchReport(rp.ReportMeta("ndgx-0.1", "00ff12ab34cd56ef", "2026-10-17T00:00:00Z"), _rows())
    ours = rp.report_to_csv(rep)
    assert _ref_roundtrip(tmp_path, ours) == ours


def test_timing_row_is_base_row_plus_fill_stats():
    mesh = ndgx.Mesh(2, (40, 30), 8)
    cfg = ndgx.SolverConfig(mesh, ndgx.EquationModel.isothermal_euler(2, 1.0), ndgx.RK4, 0.4, 1.0)
    st = ndgx.StepStats(10, 1e-3, 2e-3, 0.5)
    row = rp.timing_row(cfg, st, 1, "B200", nk=5, seed=9)
    assert (row.equation, row.rk, row.nx, row.ny, row.nz, row.nk, row.seed) == ("euler", "rk4", 40, 30, 0, 0, 0)
    assert row.dof == 40 * 30 * 64 * 3 and math.isnan(row.t_end)
    assert row.time_per_dof == 0.5 / row.dof and row.steps == 10


@pytest.mark.gpu
def test_gpu_timing_rows_read_back_by_the_reference(tmp_path):
    rows = []
    for dim, cells, order, euler, rk in [(2, (16, 12), 8, True, ndgx.RK4), (3, (4, 4, 4), 4, True, ndgx.RK6),
                                         (1, (64,), 5, False, ndgx.RK3)]:
        mesh = ndgx.Mesh(dim, cells, order)
        model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if euler else ndgx.EquationModel.advection(dim, (1,))
        cfg = ndgx.SolverConfig(mesh, model, rk, 0.4, 1.0)
        u0 = ndgx.init_euler_subsonic(mesh, model) if euler else ndgx.init_multisine(mesh, model, n_modes=3, seed=4)
        with ndgx.Solver(cfg) as s:
            s.upload(u0)
            st = s.advance(ndgx.StepPlan(4, True))
        rows.append(rp.timing_row(cfg, st, 1, "B200", nk=3, seed=4))
        assert rows[-1].steps == 4 and rows[-1].wall_seconds > 0
    ours = rp.report_to_csv(rp.BenchReport(rows=rows))
    if os.path.exists(REF_REPORT):
        assert _ref_roundtrip(tmp_path, ours) == ours
