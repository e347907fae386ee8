"""Benchmark rows in the reference's report schema.

The reference's experiment drivers (run_timing / run_scale,
src/experiments.cpp:270-399) write BenchRow records through report_to_csv
(src/report.cpp:71-120, 180-198): a two-line "# ndg-bench report" header,
the fixed column order of include/ndg/report.hpp:17-53, doubles as "%.17g"
(empty when NaN), steps empty when negative, and RFC-4180 quoting.  This
module writes the same bytes for GPU rows, so ndgx timings drop straight
into the reference's reports and plots.  tests/test_report.py pins the
output against the reference's own reader and writer.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, fields
from typing import List

NAN = float("nan")

# include/ndg/report.hpp:17-53 / src/report.cpp:71-120 (order matters)
COLUMNS = ["experiment", "row_type", "status", "equation", "dim", "order", "rk", "nx", "ny", "nz", "nk", "seed",
           "cfl", "t_end", "workers", "steps", "dof", "dt_min", "dt_max", "wall_seconds", "time_per_dof",
           "l2_error", "slope", "target_error", "fit_c", "fit_c_ref", "speedup", "efficiency", "device",
           "power_watts", "energy_joules", "energy_per_dof", "note"]


@dataclass
class BenchRow:
    experiment: str = ""
    row_type: str = "run"
    status: str = "ok"
    equation: str = ""
    rk: str = ""
    device: str = ""
    note: str = ""
    dim: int = 0
    order: int = 0
    nx: int = 0
    ny: int = 0
    nz: int = 0
    nk: int = 0
    workers: int = 0
    seed: int = 0
    cfl: float = NAN
    t_end: float = NAN
    steps: int = -1
    dof: int = 0
    dt_min: float = NAN
    dt_max: float = NAN
    wall_seconds: float = NAN
    time_per_dof: float = NAN
    l2_error: float = NAN
    slope: float = NAN
    target_error: float = NAN
    fit_c: float = NAN
    fit_c_ref: float = NAN
    speedup: float = NAN
    efficiency: float = NAN
    power_watts: float = NAN
    energy_joules: float = NAN
    energy_per_dof: float = NAN


@dataclass
class ReportMeta:
    version: str = "ndgx"
    config_digest: str = ""
    timestamp: str = ""


@dataclass
class BenchReport:
    meta: ReportMeta = field(default_factory=ReportMeta)
    rows: List[BenchRow] = field(default_factory=list)


_DOUBLES = {f.name for f in fields(BenchRow) if f.type in ("float", float)}


def fmt_double(v: float) -> str:
    """fmt_double (src/report.cpp:32-36): "%.17g"; NaN -> empty (dbl_col)."""
    return "" if math.isnan(v) else "%.17g" % v


def _cell(row: BenchRow, name: str) -> str:
    v = getattr(row, name)
    if name in _DOUBLES:
        return fmt_double(v)
    if name == "steps":
        return "" if v < 0 else str(v)
    return str(v)


def csv_escape(s: str) -> str:
    """csv_escape (src/report.cpp:122-131)."""
    if not any(ch in s for ch in ',"\n'):
        return s
    return '"' + s.replace('"', '""') + '"'


def report_to_csv(report: BenchReport) -> str:
    """report_to_csv (src/report.cpp:180-198)."""
    out = ["# ndg-bench report\n",
           f"# version={report.meta.version} config={report.meta.config_digest} timestamp={report.meta.timestamp}\n",
           ",".join(COLUMNS) + "\n"]
    for row in report.rows:
        out.append(",".join(csv_escape(_cell(row, c)) for c in COLUMNS) + "\n")
    return "".join(out)


RK_NAMES = ("rk3", "rk4", "rk6")  # rk_name (src/solver.cpp:132-139), indexed by RK3/RK4/RK6


def timing_row(cfg, stats, workers: int, device: str, experiment: str = "timing", nk: int = 0, seed: int = 0,
               note: str = "") -> BenchRow:
    """One run row as the reference's drivers build it: base_row + fill_stats
    (src/experiments.cpp:50-75).  `cfg` is a SolverConfig, `stats` the
    StepStats of the run (wall_seconds from CUDA events)."""
    mesh, model = cfg.mesh, cfg.model
    advection = model.kind == 0
    row = BenchRow(experiment=experiment, equation="advection" if advection else "euler", dim=mesh.dim,
                   order=mesh.order, rk=RK_NAMES[cfg.rk], nx=mesh.cells[0], ny=mesh.cells[1] if mesh.dim > 1 else 0,
                   nz=mesh.cells[2] if mesh.dim > 2 else 0, nk=nk if advection else 0,
                   seed=seed if advection else 0, cfl=cfg.cfl, workers=workers, dof=mesh.dof(model), device=device,
                   note=note)
    row.steps = int(stats.steps)
    row.dt_min = stats.dt_min
    row.dt_max = stats.dt_max
    row.wall_seconds = stats.wall_seconds
    row.time_per_dof = stats.wall_seconds / float(row.dof)
    return row


def scale_row(cfg, stats, workers: int, device: str, mode: str, baseline_wall: float = 0.0,
              baseline_tpd: float = 0.0, note: str = "") -> BenchRow:
    """One run_scale row (src/experiments.cpp:306-399): base_row + fill_stats
    with note = mode ("strong" / "weak"); a strong row against the serial
    baseline's wall time gets speedup = baseline_wall / wall and efficiency =
    speedup / workers, a weak row efficiency = baseline_tpd / time_per_dof
    (baseline = the 1-worker row of the same mode)."""
    row = timing_row(cfg, stats, workers, device, experiment="scale", note=mode + (f" ({note})" if note else ""))
    if baseline_wall > 0.0:
        row.speedup = baseline_wall / row.wall_seconds
        row.efficiency = row.speedup / workers
    if baseline_tpd > 0.0:
        row.efficiency = baseline_tpd / row.time_per_dof
    return row
