"""Experiment drivers on the GPU path.

The reference's sweeps (src/experiments.cpp) call one function per run,
timed_run (src/experiments.cpp:82-90); here that call goes through the ndgx
solver on a B200, and everything around it -- the spec, the row builders,
the log-log slope and the dof-for-error interpolation -- follows the
reference line for line, so a report from these drivers is the reference's
report with GPU timings.  With ``arith=ARITH_EXACT`` (the default here) the
states are bit-identical to the reference's, and so are the L2 errors,
slopes and fit constants: tests/test_experiments.py checks whole reports
against the reference's own run_converge / run_fit / run_timing.

Rows with workers > 1 go through run_partitioned (src/partition.cpp:186-333,
timed_run's own multi-worker branch): the worker count's decompose() blocks
in one partitioned handle, block w on devices[w % len(devices)].  A worker
count the mesh cannot be decomposed into gets the reference's "skipped" row
(DecompositionError); a failing run its "failed" row.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

from . import ndgx
from .report import BenchReport, BenchRow, ReportMeta


@dataclass
class DeviceProfile:
    """DeviceProfile (include/ndg/experiments.hpp)."""
    name: str
    watts: float = 0.0


@dataclass
class ExperimentSpec:
    """ExperimentSpec (include/ndg/experiments.hpp); same defaults."""
    experiment: str = "converge"
    equation: str = "advection"
    dim: int = 1
    orders: List[int] = field(default_factory=lambda: [4])
    rk: str = "rk6"
    cells: List[int] = field(default_factory=list)
    nk: int = 4
    seed: int = 0
    workers: List[int] = field(default_factory=lambda: [1])
    cfl: float = 0.4
    t_end: float = 1.0
    steps: int = 100
    devices: List[DeviceProfile] = field(default_factory=list)
    compare_equations: bool = False
    dim_compare: bool = False
    dump_path: str = ""


def _g6(x: float) -> str:
    """std::ostream default formatting of a double (precision 6, %g)."""
    return "%g" % x


def canonical_spec_string(spec: ExperimentSpec) -> str:
    """canonical_spec_string (src/experiments.cpp:155-172)."""
    j = lambda xs: ",".join(str(x) for x in xs)  # noqa: E731
    devs = ",".join(f"{d.name}:{_g6(d.watts)}" for d in spec.devices)
    return (f"experiment={spec.experiment};equation={spec.equation};dim={spec.dim};orders={j(spec.orders)}"
            f";rk={spec.rk};cells={j(spec.cells)};nk={spec.nk};seed={spec.seed};workers={j(spec.workers)}"
            f";cfl={_g6(spec.cfl)};t_end={_g6(spec.t_end)};steps={spec.steps};devices={devs}"
            f";compare_equations={int(spec.compare_equations)};dim_compare={int(spec.dim_compare)}")


def hex_digest64(text: str) -> str:
    """hex_digest64 (src/report.cpp:284-293): FNV-1a 64 over the bytes."""
    h = 0xCBF29CE484222325
    for ch in text.encode():
        h = ((h ^ ch) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def new_report(spec: ExperimentSpec) -> BenchReport:
    """new_report (src/experiments.cpp:42-48)."""
    meta = ReportMeta(ndgx.version().split()[1], hex_digest64(canonical_spec_string(spec)),
                      time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()))
    return BenchReport(meta, [])


def spec_model(spec: ExperimentSpec, dim: int) -> ndgx.EquationModel:
    """spec_model (src/experiments.cpp:20-28)."""
    if spec.equation == "advection":
        return ndgx.EquationModel.advection(dim, (1.0, 0.0, 0.0))
    if spec.equation == "euler":
        return ndgx.EquationModel.isothermal_euler(dim, 1.0)
    raise ndgx.ConfigError(f"unknown equation '{spec.equation}' (advection or euler)")


def spec_mesh(dim: int, cells_per_axis: int, order: int) -> ndgx.Mesh:
    """spec_mesh (src/experiments.cpp:30-32)."""
    return ndgx.Mesh(dim, (cells_per_axis,) * dim, order)


def spec_initial(spec: ExperimentSpec, mesh: ndgx.Mesh, model: ndgx.EquationModel):
    """spec_initial (src/experiments.cpp:34-40)."""
    if model.kind == ndgx.ADVECTION:
        return ndgx.init_multisine(mesh, model, n_modes=spec.nk, seed=spec.seed)
    return ndgx.init_euler_subsonic(mesh, model)


def base_row(spec: ExperimentSpec, mesh: ndgx.Mesh, model: ndgx.EquationModel, workers: int) -> BenchRow:
    """base_row (src/experiments.cpp:50-67)."""
    adv = model.kind == ndgx.ADVECTION
    return BenchRow(experiment=spec.experiment, equation=spec.equation, dim=mesh.dim, order=mesh.order,
                    rk=spec.rk, nx=mesh.cells[0], ny=mesh.cells[1] if mesh.dim > 1 else 0,
                    nz=mesh.cells[2] if mesh.dim > 2 else 0, nk=spec.nk if adv else 0,
                    seed=spec.seed if adv else 0, cfl=spec.cfl, workers=workers, dof=mesh.dof(model))


def fill_stats(row: BenchRow, stats: ndgx.StepStats) -> None:
    """fill_stats (src/experiments.cpp:69-75)."""
    row.steps = int(stats.steps)
    row.dt_min = stats.dt_min
    row.dt_max = stats.dt_max
    row.wall_seconds = stats.wall_seconds
    row.time_per_dof = stats.wall_seconds / float(row.dof)


@dataclass
class Runner:
    """Where timed_run's solves go: GPUs ``devices`` (default [device]), in ``arith`` mode."""
    device: int = 0
    arith: int = ndgx.ARITH_EXACT
    devices: Optional[List[int]] = None

    def timed_run(self, config: ndgx.SolverConfig, initial, plan: ndgx.StepPlan, workers: int):
        """timed_run (src/experiments.cpp:82-90) on the GPU: advance for one
        worker, run_partitioned for more."""
        if workers <= 1:
            r = ndgx.advance(config, initial, plan, device=self.device, arith=self.arith)
            return r.state, r.stats
        r = ndgx.run_partitioned(config, initial, workers, plan, devices=self.devices or [self.device],
                                 arith=self.arith)
        return r.state, r.stats


def loglog_slope(n: List[float], err: List[float]) -> float:
    """loglog_slope (src/experiments.cpp:174-194), same summation order."""
    if len(n) != len(err) or len(n) < 2:
        return math.nan
    m = len(n)
    x = [math.log(v) for v in n]
    y = [math.log(v) for v in err]
    sx = sy = 0.0
    for i in range(m):
        sx += x[i]
        sy += y[i]
    mx, my = sx / m, sy / m
    num = den = 0.0
    for i in range(m):
        num += (x[i] - mx) * (y[i] - my)
        den += (x[i] - mx) * (x[i] - mx)
    return math.nan if den == 0.0 else num / den


def interpolate_dof_for_error(dof_and_error: List[Tuple[float, float]], target: float) -> float:
    """interpolate_dof_for_error (src/experiments.cpp:196-210)."""
    for i in range(len(dof_and_error) - 1):
        d0, e0 = dof_and_error[i]
        d1, e1 = dof_and_error[i + 1]
        if e0 >= target > e1:
            t = (math.log(target) - math.log(e0)) / (math.log(e1) - math.log(e0))
            return math.exp(math.log(d0) + t * (math.log(d1) - math.log(d0)))
    if dof_and_error and dof_and_error[0][1] <= target:
        return dof_and_error[0][0]
    return math.nan


def converge_rows(spec: ExperimentSpec, report: BenchReport, runner: Runner) -> List[BenchRow]:
    """converge_rows (src/experiments.cpp:93-121): t_end runs against the
    exact solution (the advected profile returns to the start at t=1)."""
    if spec.equation != "advection":
        raise ndgx.ConfigError(f"{spec.experiment} measures the advected profile and needs --equation advection")
    if not spec.cells:
        raise ndgx.ConfigError("empty cell sweep")
    rows = []
    for order in spec.orders:
        for c in spec.cells:
            mesh = spec_mesh(spec.dim, c, order)
            model = spec_model(spec, spec.dim)
            row = base_row(spec, mesh, model, 1)
            row.t_end = spec.t_end
            try:
                initial = spec_initial(spec, mesh, model)
                config = ndgx.SolverConfig(mesh, model, ndgx.rk_from_name(spec.rk), spec.cfl, spec.t_end)
                state, stats = runner.timed_run(config, initial, ndgx.StepPlan(-1, True), 1)
                fill_stats(row, stats)
                row.l2_error = ndgx.l2_error(mesh, model, state, initial, 0)
            except ndgx.InstabilityError as e:
                row.status = "failed"
                row.note = str(e)
            report.rows.append(row)
            rows.append(row)
    return rows


def make_slope_row(spec: ExperimentSpec, order: int, rows: List[BenchRow]) -> BenchRow:
    """make_slope_row (src/experiments.cpp:123-151)."""
    s = BenchRow(experiment=spec.experiment, row_type="slope", equation=spec.equation, dim=spec.dim, order=order,
                 rk=spec.rk, nk=spec.nk, seed=spec.seed, cfl=spec.cfl, t_end=spec.t_end)
    n, err = [], []
    for r in rows:
        if r.order == order and r.row_type == "run" and r.status == "ok" and r.l2_error > 1e-11:
            n.append(float(r.nx))
            err.append(r.l2_error)
    s.slope = loglog_slope(n, err)
    if math.isnan(s.slope):
        s.status = "skipped"
        s.note = "fewer than two points above the 1e-11 error floor"
    return s


def run_converge(spec: ExperimentSpec, runner: Optional[Runner] = None) -> BenchReport:
    """run_converge (src/experiments.cpp:212-219)."""
    runner = runner or Runner()
    report = new_report(spec)
    rows = converge_rows(spec, report, runner)
    for order in spec.orders:
        report.rows.append(make_slope_row(spec, order, rows))
    return report


def run_cost(spec: ExperimentSpec, runner: Optional[Runner] = None) -> BenchReport:
    """run_cost (src/experiments.cpp:221-225)."""
    report = new_report(spec)
    converge_rows(spec, report, runner or Runner())
    return report


def fit_rows(spec: ExperimentSpec, rows: List[BenchRow]) -> List[BenchRow]:
    """run_fit's fit rows (src/experiments.cpp:232-265): dof needed for
    1e-2/1e-3/1e-4 and the constant dof * err^(1/order) (reference 200)."""
    out = []
    for order in spec.orders:
        curve = sorted((float(r.dof), r.l2_error) for r in rows if r.order == order and r.status == "ok")
        for target in (1e-2, 1e-3, 1e-4):
            f = BenchRow(experiment=spec.experiment, row_type="fit", equation=spec.equation, dim=spec.dim,
                         order=order, rk=spec.rk, nk=spec.nk, seed=spec.seed, cfl=spec.cfl, t_end=spec.t_end,
                         target_error=target, fit_c_ref=200.0)
            need = interpolate_dof_for_error(curve, target)
            if math.isnan(need):
                f.status = "unreachable"
                f.note = "target error outside the measured range"
            else:
                f.dof = _llround(need)
                f.fit_c = need * math.pow(target, 1.0 / order)
                if curve and curve[0][1] <= target:
                    f.note = "coarsest grid already meets the target; dof is an upper bound"
            out.append(f)
    return out


def run_fit(spec: ExperimentSpec, runner: Optional[Runner] = None) -> BenchReport:
    """run_fit (src/experiments.cpp:227-268)."""
    report = new_report(spec)
    rows = converge_rows(spec, report, runner or Runner())
    report.rows.extend(fit_rows(spec, rows))
    return report


def _llround(x: float) -> int:
    """std::llround: half away from zero."""
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def run_timing(spec: ExperimentSpec, runner: Optional[Runner] = None) -> BenchReport:
    """run_timing (src/experiments.cpp:270-304): fixed-step warm runs."""
    runner = runner or Runner()
    report = new_report(spec)
    if not spec.cells:
        raise ndgx.ConfigError("empty cell sweep")
    equations = [spec.equation]
    if spec.compare_equations:
        equations.append("euler" if spec.equation == "advection" else "advection")
    workers = spec.workers[0] if spec.workers else 1
    for eq in equations:
        eq_spec = ExperimentSpec(**{**spec.__dict__, "equation": eq})
        for order in spec.orders:
            for c in spec.cells:
                mesh = spec_mesh(spec.dim, c, order)
                model = spec_model(eq_spec, spec.dim)
                row = base_row(eq_spec, mesh, model, workers)
                try:
                    initial = spec_initial(eq_spec, mesh, model)
                    config = ndgx.SolverConfig(mesh, model, ndgx.rk_from_name(spec.rk), spec.cfl, spec.t_end)
                    _, stats = runner.timed_run(config, initial, ndgx.StepPlan(spec.steps, True), workers)
                    fill_stats(row, stats)
                except ndgx.DecompositionError as e:
                    row.status = "skipped"
                    row.note = str(e)
                except RuntimeError as e:
                    row.status = "failed"
                    row.note = str(e)
                report.rows.append(row)
    return report


def weak_grid(dim: int, cells: int, p: int) -> Tuple[int, int, int]:
    """run_scale's weak-scaling factorisation (src/experiments.cpp:352-378): the
    lowest-interface (px, py, pz) of p workers for c cells per worker per axis,
    ties broken by the lexicographically smallest grid."""
    best, best_cost = (1, 1, 1), -1
    for px in range(1, p + 1):
        if p % px:
            continue
        rest = p // px
        for py in range(1, rest + 1):
            if rest % py:
                continue
            pz = rest // py
            if dim < 3 and pz != 1:
                continue
            if dim < 2 and py != 1:
                continue
            grid = (px, py, pz)
            cost = 0
            for d in range(dim):
                cross = 1
                for e in range(dim):
                    if e != d:
                        cross *= cells * grid[e]
                cost += grid[d] * cross
            if best_cost < 0 or cost < best_cost or (cost == best_cost and grid < best):
                best, best_cost = grid, cost
    return best


def run_scale(spec: ExperimentSpec, runner: Optional[Runner] = None) -> BenchReport:
    """run_scale (src/experiments.cpp:306-399): per cell count, strong scaling
    of the fixed grid against its 1-worker wall time, then weak scaling on the
    lowest-interface grid of c cells per worker per axis against the 1-worker
    time per DOF.  Multi-worker rows run through the partitioned handle
    (Runner.devices: block w on devices[w % len]); on one GPU every block
    shares it, so the speedup column measures the decomposition's cost there,
    not a multi-GPU speedup (bench.py under torchrun gives those)."""
    runner = runner or Runner()
    report = new_report(spec)
    if not spec.cells:
        raise ndgx.ConfigError("empty cell sweep")
    if spec.dim < 2:
        raise ndgx.ConfigError("scaling runs need dim >= 2")
    if spec.dim_compare:
        raise ndgx.ConfigError("--dim-compare is not on the GPU path (SURVEY.md §8)")
    order = spec.orders[0]

    def run_one(mesh, workers, mode, baseline_wall, baseline_tpd):
        model = spec_model(spec, spec.dim)
        row = base_row(spec, mesh, model, workers)
        row.note = mode
        try:
            initial = spec_initial(spec, mesh, model)
            config = ndgx.SolverConfig(mesh, model, ndgx.rk_from_name(spec.rk), spec.cfl, spec.t_end)
            _, stats = runner.timed_run(config, initial, ndgx.StepPlan(spec.steps, True), workers)
            fill_stats(row, stats)
            if baseline_wall > 0.0:
                row.speedup = baseline_wall / stats.wall_seconds
                row.efficiency = row.speedup / workers
            if baseline_tpd > 0.0:
                row.efficiency = baseline_tpd / row.time_per_dof
        except ndgx.DecompositionError as e:
            row.status = "skipped"
            row.note = f"{mode}: {e}"
        except RuntimeError as e:
            row.status = "failed"
            row.note = f"{mode}: {e}"
        report.rows.append(row)
        return row

    for c in spec.cells:
        glob = spec_mesh(spec.dim, c, order)
        serial = run_one(glob, 1, "strong", 0.0, 0.0)
        for p in spec.workers:
            if p <= 1:
                continue
            run_one(glob, p, "strong", serial.wall_seconds if serial.status == "ok" else 0.0, 0.0)
        weak_tpd = 0.0
        for p in spec.workers:
            g = weak_grid(spec.dim, c, p)
            cells = tuple(c * g[a] for a in range(spec.dim))
            row = run_one(ndgx.Mesh(spec.dim, cells, order), p, "weak", 0.0, weak_tpd)
            if p == 1 and row.status == "ok":
                weak_tpd = row.time_per_dof
    return report


def run_experiment(spec: ExperimentSpec, runner: Optional[Runner] = None) -> BenchReport:
    """run_experiment (src/experiments.cpp:521-531) for the sweeps on the GPU path."""
    fns = {"converge": run_converge, "cost": run_cost, "fit": run_fit, "timing": run_timing, "scale": run_scale}
    if spec.experiment not in fns:
        raise ndgx.ConfigError(f"unknown experiment '{spec.experiment}'"
                               if spec.experiment not in ("energy", "simulate") else
                               f"experiment '{spec.experiment}' is not on the GPU path (SURVEY.md §8)")
    return fns[spec.experiment](spec, runner)


def main(argv=None) -> int:
    """``python -m paper_2510_05254_b200.experiments <experiment> [options]``:
    the sweep options of the reference's ndg-bench (tools/ndg_bench.cpp:72-98)
    for the experiments on the GPU path; CSV reports only."""
    import argparse
    ap = argparse.ArgumentParser(prog="python -m paper_2510_05254_b200.experiments")
    ap.add_argument("experiment", choices=["converge", "cost", "fit", "timing", "scale"])
    ap.add_argument("--equation", default="advection")
    ap.add_argument("--dim", type=int, default=1)
    ap.add_argument("--order", type=int, action="append")
    ap.add_argument("--rk", default="rk6")
    ap.add_argument("--cells", type=int, action="append")
    ap.add_argument("--nk", type=int, default=4)
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--workers", type=int, action="append")
    ap.add_argument("--cfl", type=float, default=0.4)
    ap.add_argument("--t-end", type=float, default=1.0)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--compare-equations", action="store_true")
    ap.add_argument("--arith", choices=["exact", "fast"], default="exact")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--devices", type=int, action="append",
                    help="GPUs of the multi-worker rows (block w on devices[w %% len]); default [--device]")
    ap.add_argument("--out", default=None, help="report path (default: <experiment>.csv)")
    a = ap.parse_args(argv)
    if a.equation == "advection" and a.seed is None:
        ap.error("--seed is required for experiments with random sine amplitudes")
    if not a.cells:
        ap.error("--cells is required (one value per run in the sweep)")
    spec = ExperimentSpec(a.experiment, a.equation, a.dim, a.order or [4], a.rk, a.cells, a.nk, a.seed or 0,
                          a.workers or [1], a.cfl, a.t_end, a.steps, compare_equations=a.compare_equations)
    rep = run_experiment(spec, Runner(a.device, ndgx.ARITH_FAST if a.arith == "fast" else ndgx.ARITH_EXACT,
                                      a.devices))
    from .report import report_to_csv
    with open(a.out or f"{a.experiment}.csv", "w") as f:
        f.write(report_to_csv(rep))
    return 1 if any(r.status == "failed" for r in rep.rows) else 0


if __name__ == "__main__":
    raise SystemExit(main())
