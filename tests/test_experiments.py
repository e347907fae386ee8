"""Experiment sweeps on the GPU path.

Pins: the reference's own run_experiment (tests/cpp/ref_experiments, built
from src/experiments.cpp + src/report.cpp over oracle/_ref) on the CPU.  The
CPU tests check the host logic (spec digest, slope and fit rows, l2_error /
conserved_totals) against it; the GPU tests run whole sweeps through the
B200 solver in exact mode and require every column of the report except the
wall-clock ones to match the reference's bytes.  The acceptance criteria
C1/C2/C8 (proj/tests/acceptance.cpp:73-115, 340-394) are then evaluated at
sizes the CPU reference is not run at.
"""
from __future__ import annotations

import math
import os
import subprocess

import numpy as np
import pytest

import paper_2510_05254_b200 as ndgx
from paper_2510_05254_b200 import experiments as ex
from paper_2510_05254_b200 import report as rp

REF_EXP = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "ref_experiments")
TIMING_COLS = {"wall_seconds", "time_per_dof", "speedup", "efficiency"}  # measured, not computed from states


def _ref_csv(spec: ex.ExperimentSpec) -> str:
    if not os.path.exists(REF_EXP):
        pytest.skip("tests/cpp/_build/ref_experiments not built (needs /root/reference at build time)")
    args = [spec.experiment, spec.equation, str(spec.dim), ",".join(map(str, spec.orders)), spec.rk,
            ",".join(map(str, spec.cells)), str(spec.nk), str(spec.seed), ",".join(map(str, spec.workers)),
            repr(spec.cfl), repr(spec.t_end), str(spec.steps), str(int(spec.compare_equations))]
    return subprocess.run([REF_EXP, *args], check=True, capture_output=True, text=True, timeout=300).stdout


def _parse(csv: str):
    lines = csv.splitlines()
    meta = dict(tok.split("=", 1) for tok in lines[1][2:].split())
    cols = lines[2].split(",")
    return meta, [dict(zip(cols, ln.split(","))) for ln in lines[3:]]


def _rows_from_ref(rows):
    """BenchRows rebuilt from the reference's CSV cells (for the host-logic checks)."""
    out = []
    for r in rows:
        b = rp.BenchRow(experiment=r["experiment"], row_type=r["row_type"], status=r["status"],
                        order=int(r["order"]), nx=int(r["nx"]), dof=int(r["dof"]))
        b.l2_error = float(r["l2_error"]) if r["l2_error"] else math.nan
        out.append(b)
    return out


SPECS = [
    ex.ExperimentSpec("converge", "advection", 1, [3, 4, 6], "rk6", [4, 8, 16, 32], 4, 42),
    ex.ExperimentSpec("fit", "advection", 1, [3, 5], "rk4", [8, 16, 32, 64], 7, 3),
    ex.ExperimentSpec("converge", "advection", 2, [4], "rk3", [4, 8], 3, 11, cfl=0.3, t_end=0.5),
    ex.ExperimentSpec("timing", "euler", 2, [8], "rk4", [6, 8], steps=12, compare_equations=True),
    # run_scale: strong rows of an 8^2 grid at 1/2/4 workers, weak rows on the
    # lowest-interface grids (multi-worker rows through the partitioned handle)
    ex.ExperimentSpec("scale", "euler", 2, [4], "rk4", [8], workers=[1, 2, 4], steps=5),
    ex.ExperimentSpec("scale", "advection", 3, [3], "rk3", [4], 3, 5, workers=[1, 3], steps=4),
]


# ------------------------------------------------------------------ CPU
@pytest.mark.parametrize("spec", SPECS, ids=lambda s: f"{s.experiment}-{s.dim}d")
def test_config_digest_matches_the_reference(spec):
    meta, _ = _parse(_ref_csv(spec))
    assert ex.hex_digest64(ex.canonical_spec_string(spec)) == meta["config"]
    assert meta["version"] == ndgx.version().split()[1]


@pytest.mark.parametrize("spec", SPECS[:2], ids=lambda s: s.experiment)
def test_slope_and_fit_rows_from_the_reference_runs(spec):
    """make_slope_row / run_fit's rows recomputed from the reference's own run
    rows must be the reference's rows, byte for byte."""
    _, ref = _parse(_ref_csv(spec))
    runs = [r for r in ref if r["row_type"] == "run"]
    rows = _rows_from_ref(runs)
    if spec.experiment == "converge":
        got = [ex.make_slope_row(spec, order, rows) for order in spec.orders]
    else:
        got = ex.fit_rows(spec, rows)
    want = [r for r in ref if r["row_type"] != "run"]
    mine = _parse(rp.report_to_csv(rp.BenchReport(rows=got)))[1]
    assert mine == want


def test_loglog_slope_and_interpolation_edges():
    assert math.isnan(ex.loglog_slope([4.0], [1e-3]))
    assert math.isnan(ex.loglog_slope([4.0, 4.0], [1e-3, 1e-4]))
    assert ex.loglog_slope([1.0, 2.0], [1.0, 0.25]) == pytest.approx(-2.0, abs=1e-15)
    assert math.isnan(ex.interpolate_dof_for_error([(10.0, 1e-2), (20.0, 5e-3)], 1e-4))
    assert ex.interpolate_dof_for_error([(10.0, 1e-5), (20.0, 1e-6)], 1e-4) == 10.0
    assert ex.interpolate_dof_for_error([(10.0, 1e-2), (100.0, 1e-4)], 1e-3) == pytest.approx(10 ** 1.5)
    assert ex._llround(2.5) == 3 and ex._llround(-2.5) == -3


@pytest.mark.parametrize("dim,cells,order,euler", [(1, (9,), 5, False), (2, (5, 3), 8, True), (3, (3, 2, 2), 4, True)])
def test_l2_error_and_totals_bit_identical_to_the_reference(reference, dim, cells, order, euler):
    from oracle_lib import ADVECTION, EULER, Problem
    mesh = ndgx.Mesh(dim, cells, order, tuple(0.5 + a for a in range(dim)))
    model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if euler else ndgx.EquationModel.advection(dim, (1,))
    p = Problem(dim, cells, order, EULER if euler else ADVECTION, length=tuple(mesh.length) + (1.0,) * (3 - dim))
    rng = np.random.default_rng(dim)
    a, b = rng.standard_normal((2, mesh.dof(model)))
    for v in range(model.n_var()):
        assert ndgx.l2_error(mesh, model, a, b, v) == reference.l2_error(p, a, b, v)
    assert np.array_equal(ndgx.conserved_totals(mesh, model, a), reference.conserved_totals(p, a))
    with pytest.raises(IndexError):
        ndgx.l2_error(mesh, model, a, b, model.n_var())


def test_multi_worker_timing_rows_skip_undecomposable_meshes():
    # timed_run's multi-worker branch is run_partitioned: a worker count the
    # mesh cannot be split into is the reference's "skipped" row (decided on
    # the host, before any device work)
    spec = ex.ExperimentSpec("timing", "euler", 2, [4], "rk4", [1], workers=[3], steps=2)
    rows = ex.run_timing(spec, ex.Runner()).rows
    assert [r.status for r in rows] == ["skipped"] and rows[0].workers == 3


def test_energy_and_simulate_drivers_are_not_on_the_gpu_path():
    for name in ("energy", "simulate"):
        with pytest.raises(ndgx.ConfigError, match="not on the GPU path"):
            ex.run_experiment(ex.ExperimentSpec(name))


def test_weak_grid_is_the_references_lowest_interface_factorisation():
    # src/experiments.cpp:352-378: ties go to the lexicographically smallest grid
    assert ex.weak_grid(2, 8, 1) == (1, 1, 1)
    assert ex.weak_grid(2, 8, 2) == (1, 2, 1)
    assert ex.weak_grid(2, 8, 4) == (1, 4, 1)
    assert ex.weak_grid(2, 8, 6) == (1, 6, 1)
    assert ex.weak_grid(3, 4, 8) == (1, 1, 8)
    assert ex.weak_grid(3, 4, 3) == (1, 1, 3)
    with pytest.raises(ndgx.ConfigError, match="scaling runs need dim >= 2"):
        ex.run_scale(ex.ExperimentSpec("scale", "advection", 1, [3], "rk3", [4], 3, 5))


@pytest.mark.gpu
def test_multi_worker_timing_rows_run_partitioned():
    # workers = 2: the partitioned handle; states bit-identical to one worker,
    # so every non-timing column equals the single-worker row
    one = ex.run_timing(ex.ExperimentSpec("timing", "euler", 2, [4], "rk4", [6], steps=3)).rows[0]
    two = ex.run_timing(ex.ExperimentSpec("timing", "euler", 2, [4], "rk4", [6], workers=[2], steps=3)).rows[0]
    assert two.status == "ok" and two.workers == 2
    assert (two.steps, two.dt_min, two.dt_max, two.dof) == (one.steps, one.dt_min, one.dt_max, one.dof)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("spec", SPECS, ids=lambda s: f"{s.experiment}-{s.dim}d")
def test_gpu_report_equals_the_reference_report(spec):
    ours = rp.report_to_csv(ex.run_experiment(spec))
    m0, want = _parse(_ref_csv(spec))
    m1, got = _parse(ours)
    assert (m0["version"], m0["config"]) == (m1["version"], m1["config"])
    assert len(got) == len(want)
    for g, w in zip(got, want):
        for c in rp.COLUMNS:
            if c in TIMING_COLS and w["row_type"] == "run":
                assert (g[c] == "") == (w[c] == "")
            else:
                assert g[c] == w[c], (c, g, w)


def _doubling_slopes(cells, errors, floor=1e-11):
    """doubling_slopes (proj/tests/acceptance.cpp:59-69)."""
    return [math.log2(errors[i] / errors[i + 1]) / math.log2(cells[i + 1] / cells[i])
            for i in range(len(errors) - 1) if errors[i] > floor and errors[i + 1] > floor]


def _errors(dim, order, rk, cells, nk=4, seed=42):
    spec = ex.ExperimentSpec("converge", "advection", dim, [order], rk, cells, nk, seed)
    return [r.l2_error for r in ex.run_converge(spec).rows if r.row_type == "run"]


@pytest.mark.gpu
def test_c1_spatial_convergence_on_gpu():
    """Criterion 1 (acceptance.cpp:73-95): best doubling slope >= order - 0.5,
    orders 3..8, 4..256 cells, RK6 (runtime limit there: 120 s on the CPU)."""
    cells = [4, 8, 16, 32, 64, 128, 256]
    for order in range(3, 9):
        best = max(_doubling_slopes(cells, _errors(1, order, "rk6", cells)))
        assert best >= order - 0.5, (order, best)


@pytest.mark.gpu
def test_c2_temporal_order_reduction_on_gpu():
    """Criterion 2 (acceptance.cpp:97-115): RK3 fine slope 3 +- 0.4, RK6 >= 5.5."""
    cells = [8, 16, 32, 64, 128, 256]
    s3 = _doubling_slopes(cells, _errors(1, 6, "rk3", cells))
    s6 = _doubling_slopes(cells, _errors(1, 6, "rk6", cells))
    assert abs(s3[-1] - 3.0) <= 0.4 and min(s6) >= 5.5, (s3, s6)


@pytest.mark.gpu
def test_2d_order8_convergence_at_gpu_scale():
    """2D advection, order 8, up to 128^2 cells (1M DOF, t_end = 1): the
    sweep converges at the design order until the error floor."""
    cells = [4, 8, 16, 32, 64, 128]
    errs = _errors(2, 8, "rk6", cells)
    slopes = _doubling_slopes(cells, errs)
    assert max(slopes) >= 7.5, (errs, slopes)


@pytest.mark.gpu
def test_c8_fit_constants_on_gpu():
    """Criterion 8 (acceptance.cpp:340-394): dof * err^(1/order) at 1e-3 and
    1e-4, orders 3..8, 1D RK6 sweeps: spread <= 3x, all within 3x of 200."""
    sweeps = {3: [800, 1600, 2400], 4: [200, 400, 800], 5: [120, 240, 480], 6: [80, 160, 320],
              7: [40, 60, 120], 8: [40, 50, 100]}
    cs = []
    for order, cells in sweeps.items():
        spec = ex.ExperimentSpec("converge", "advection", 1, [order], "rk6", cells, 40, 42)
        curve = [(float(c * order), r.l2_error) for c, r in
                 zip(cells, [r for r in ex.run_converge(spec).rows if r.row_type == "run"])]
        for target in (1e-3, 1e-4):
            dof = ex.interpolate_dof_for_error(curve, target)
            assert not math.isnan(dof), (order, target, curve)
            cs.append(dof * target ** (1.0 / order))
    assert max(cs) / min(cs) <= 3.0 and max(cs) <= 600.0 and min(cs) >= 200.0 / 3.0, cs


def test_cli_writes_the_report(tmp_path, monkeypatch):
    """The CLI builds the spec like ndg-bench; the runner is stubbed (no GPU)."""
    seen = {}

    def fake(spec, runner=None):
        seen["spec"] = spec
        return rp.BenchReport(rows=[rp.BenchRow(experiment=spec.experiment)])
    monkeypatch.setattr(ex, "run_experiment", fake)
    out = tmp_path / "r.csv"
    assert ex.main(["converge", "--order", "4", "--order", "6", "--cells", "8", "--cells", "16", "--seed", "42",
                    "--out", str(out)]) == 0
    assert seen["spec"].orders == [4, 6] and seen["spec"].cells == [8, 16] and seen["spec"].seed == 42
    assert out.read_text().startswith("# ndg-bench report\n")
