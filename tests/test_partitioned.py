"""run_partitioned on the GPU: one handle over P decompose() blocks.

The reference's run_partitioned (src/partition.cpp:186-333) is bitwise equal
to its serial advance for every worker count (proj/tests/test_partition.cpp:
267-328; acceptance C6).  ndgx_create_partitioned runs the same blocks in one
handle on one B200: every block packs the stage-input planes of its split
axes straight into its neighbours' halo buffers, the interior elements run
while they land and the boundary shell after.  These tests run split blocks
(block offset != 0, planes from a different block) and check them bit for bit
against the single-block solver and the reference library's own
run_partitioned, including t_end landing and the RunError contract.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2510_05254_b200 as ndgx
from oracle_lib import ADVECTION, EULER, Problem

pytestmark = pytest.mark.gpu


def _cfg(dim, cells, order, euler, rk=ndgx.RK4, t_end=1.0):
    mesh = ndgx.Mesh(dim, cells, order)
    model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if euler else ndgx.EquationModel.advection(dim, (1, 0, 0))
    return ndgx.SolverConfig(mesh, model, rk, 0.4, t_end)


def _u0(cfg):
    if cfg.model.kind == ndgx.EULER_ISOTHERMAL:
        return ndgx.init_euler_subsonic(cfg.mesh, cfg.model)
    return ndgx.init_multisine(cfg.mesh, cfg.model, n_modes=5, seed=3)


def _problem(cfg):
    return Problem(cfg.mesh.dim, tuple(cfg.mesh.cells[:cfg.mesh.dim]), cfg.mesh.order,
                   EULER if cfg.model.kind == ndgx.EULER_ISOTHERMAL else ADVECTION, cfg.rk,
                   t_end=cfg.t_end)


# (name, (dim, cells, order, euler, rk), workers, expected decompose() grid)
CASES = [
    ("2D Euler o8 RK4 y-split", (2, (8, 16), 8, True, ndgx.RK4), 2, (1, 2, 1)),
    ("2D Euler o8 RK4 2x2", (2, (16, 16), 8, True, ndgx.RK4), 4, (2, 2, 1)),
    ("3D Euler o4 RK6 z-slabs", (3, (4, 4, 16), 4, True, ndgx.RK6), 4, (1, 1, 4)),
    ("2D adv o3 RK3 x-split", (2, (9, 7), 3, False, ndgx.RK3), 3, (3, 1, 1)),
    ("1D adv o4 RK4", (1, (64,), 4, False, ndgx.RK4), 4, (4, 1, 1)),
    ("2D adv o8 RK4 2x2", (2, (12, 12), 8, False, ndgx.RK4), 4, (2, 2, 1)),
    ("2D Euler o7 RK4 2x2 (padded body)", (2, (10, 12), 7, True, ndgx.RK4), 4, (2, 2, 1)),
    ("2D Euler o6 RK3 x-split (padded body)", (2, (12, 5), 6, True, ndgx.RK3), 2, (2, 1, 1)),
    ("2D adv o5 RK6 y-split (padded body)", (2, (6, 12), 5, False, ndgx.RK6), 2, (1, 2, 1)),
]


def _single(cfg, u0, plan, arith):
    with ndgx.Solver(cfg, arith=arith) as s:
        s.upload(u0)
        r = s.rhs()
        st = s.advance(plan)
        return r, s.download(), st


def _part(cfg, u0, workers, plan, arith, force=False):
    with ndgx.Solver.partitioned(cfg, workers, arith=arith, force_exchange=force) as s:
        grid = tuple(s.block(0).grid)
        blocks = [s.block(w) for w in range(workers)]
        s.upload(u0)
        r = s.rhs()
        st = s.advance(plan)
        return r, s.download(), st, grid, blocks


@pytest.mark.parametrize("arith", [ndgx.ARITH_EXACT, ndgx.ARITH_FAST], ids=["exact", "fast"])
@pytest.mark.parametrize("name,case,workers,grid", CASES, ids=[c[0] for c in CASES])
def test_partitioned_bitwise_equals_single_block(name, case, workers, grid, arith):
    dim, cells, order, euler, rk = case
    cfg = _cfg(dim, cells, order, euler, rk)
    u0 = _u0(cfg)
    plan = ndgx.StepPlan(7, True)
    r_want, want, st_want = _single(cfg, u0, plan, arith)
    r_got, got, st, g, blocks = _part(cfg, u0, workers, plan, arith)
    assert g == grid, f"{name}: decompose grid {g}"
    assert any(b.lo[a] != 0 for b in blocks for a in range(3)), "some block sits at a non-zero offset"
    assert np.array_equal(r_got, r_want), f"{name}: partitioned rhs differs"
    assert np.array_equal(got, want), f"{name}: partitioned state differs"
    assert (st.steps, st.dt_min, st.dt_max) == (st_want.steps, st_want.dt_min, st_want.dt_max)


@pytest.mark.parametrize("name,case,workers,grid", CASES[:3], ids=[c[0] for c in CASES[:3]])
def test_partitioned_matches_the_reference_run_partitioned(name, case, workers, grid, reference):
    dim, cells, order, euler, rk = case
    cfg = _cfg(dim, cells, order, euler, rk)
    p = _problem(cfg)
    u0 = reference.initial(p, n_modes=5, seed=3)
    want, st_want = reference.run_partitioned(p, u0, workers, 5, True)
    res = ndgx.run_partitioned(cfg, u0, workers, ndgx.StepPlan(5, True))
    assert np.array_equal(res.state, want), f"{name}: differs from the reference's run_partitioned"
    assert res.stats.steps == st_want.steps and res.stats.dt_max == st_want.dt_max
    assert len(res.worker_timings) == workers and res.decomposition.grid == grid


def test_partitioned_t_end_lands_like_the_reference(reference):
    """proj/tests/test_partition.cpp:315-328 (6x6 o3, t_end 0.03, P=2) plus a
    flagship-shaped case whose last step is shortened."""
    for cells, order, t_end, workers in (((6, 6), 3, 0.03, 2), ((16, 12), 8, 0.02, 4)):
        cfg = _cfg(2, cells, order, False, ndgx.RK4, t_end)
        p = _problem(cfg)
        u0 = reference.init_multisine(p, n_modes=3, seed=7)
        want, st_want = reference.run_partitioned(p, u0, workers, -1, False)
        res = ndgx.run_partitioned(cfg, u0, workers)
        assert res.stats.steps == st_want.steps and res.stats.dt_max == st_want.dt_max
        assert res.stats.dt_min == st_want.dt_min
        assert np.array_equal(res.state, want)


def test_partitioned_euler_t_end_fast_equals_single():
    cfg = _cfg(2, (16, 16), 8, True, ndgx.RK4, 0.02)
    u0 = _u0(cfg)
    plan = ndgx.StepPlan(-1, False)
    _, want, st_want = _single(cfg, u0, plan, ndgx.ARITH_FAST)
    _, got, st, _, _ = _part(cfg, u0, 4, plan, ndgx.ARITH_FAST)
    assert st.steps == st_want.steps and st.dt_max == st_want.dt_max
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dim,cells,order,euler,rk", [(2, (12, 10), 8, True, ndgx.RK4),
                                                      (3, (5, 4, 6), 4, True, ndgx.RK6),
                                                      (2, (7, 9), 5, False, ndgx.RK3),
                                                      (2, (9, 7), 7, True, ndgx.RK4),
                                                      (2, (6, 8), 6, True, ndgx.RK6),
                                                      (2, (1067, 3), 8, True, ndgx.RK4),
                                                      (2, (1101, 2), 8, True, ndgx.RK6)])
def test_one_worker_forced_through_the_halo_planes(dim, cells, order, euler, rk):
    """Every axis of a single block routed through its own halo planes (the
    boxes: interior + a shell on every axis) is the single-block run, also
    on 1000+-wide meshes (x-runs straddling rows, RK6 last stage)."""
    cfg = _cfg(dim, cells, order, euler, rk)
    u0 = _u0(cfg)
    plan = ndgx.StepPlan(6, False)
    for arith in (ndgx.ARITH_EXACT, ndgx.ARITH_FAST):
        r_want, want, st_want = _single(cfg, u0, plan, arith)
        r_got, got, st, _, _ = _part(cfg, u0, 1, plan, arith, force=True)
        assert np.array_equal(r_got, r_want) and np.array_equal(got, want)
        assert st.dt_max == st_want.dt_max


def test_thin_blocks_without_interior():
    """Blocks one or two cells thick along the split axis have no interior:
    the whole block is boundary shell."""
    cfg = _cfg(2, (4, 6), 6, True)
    u0 = _u0(cfg)
    plan = ndgx.StepPlan(5, False)
    _, want, _ = _single(cfg, u0, plan, ndgx.ARITH_EXACT)
    for workers in (2, 3, 6):
        _, got, _, _, _ = _part(cfg, u0, workers, plan, ndgx.ARITH_EXACT)
        assert np.array_equal(got, want), f"P={workers}"


def test_failing_worker_surfaces_as_run_error(reference):
    """proj/tests/test_partition.cpp:330-349: worker 1 owns y in [4, 8) of the
    8x8 mesh; a negative density there is RunError naming worker 1, with the
    reference's message."""
    cfg = _cfg(2, (8, 8), 3, True)
    p = _problem(cfg)
    u0 = reference.init_euler(p)
    f = u0.reshape(8, 8, 3, 3, 3)
    f[6, 6, 1, 1, 0] = -2.0
    bad = f.reshape(-1)
    with pytest.raises(Exception) as want:
        reference.run_partitioned(p, bad, 2, 4, False)
    with pytest.raises(ndgx.RunError) as got:
        ndgx.run_partitioned(cfg, bad, 2, ndgx.StepPlan(4, False))
    assert got.value.worker == 1 == want.value.worker
    assert str(got.value) == want.value.message
    assert "worker 1" in str(got.value) and "density" in str(got.value)


def test_instability_names_the_worker(reference):
    """A NaN deep inside worker 1's block: 'worker 1: non-finite state after step 1'."""
    cfg = _cfg(1, (64,), 3, False)
    p = _problem(cfg)
    u0 = reference.init_multisine(p, amps=[1.0])
    u0[48 * 3 + 1] = np.nan
    with pytest.raises(Exception) as want:
        reference.run_partitioned(p, u0, 2, 3, False)
    with pytest.raises(ndgx.RunError) as got:
        ndgx.run_partitioned(cfg, u0, 2, ndgx.StepPlan(3, False))
    assert got.value.worker == want.value.worker == 1
    assert str(got.value) == want.value.message == "worker 1: non-finite state after step 1"


def test_partitioned_checkpoint_is_the_global_field(tmp_path):
    cfg = _cfg(2, (8, 16), 8, True)
    u0 = _u0(cfg)
    with ndgx.Solver.partitioned(cfg, 2) as s:
        s.upload(u0)
        s.advance(ndgx.StepPlan(3, False))
        s.dump_field(str(tmp_path / "p.ndg"))
        got = s.download()
    with ndgx.Solver(cfg) as s:
        s.upload(u0)
        s.advance(ndgx.StepPlan(3, False))
        s.dump_field(str(tmp_path / "s.ndg"))
    assert (tmp_path / "p.ndg").read_bytes() == (tmp_path / "s.ndg").read_bytes()
    with ndgx.Solver.partitioned(cfg, 4) as s:
        s.load_field(str(tmp_path / "p.ndg"))
        assert np.array_equal(s.download(), got)


def test_partitioned_decomposition_error_is_raised():
    cfg = _cfg(2, (2, 2), 4, False)
    with pytest.raises(ndgx.DecompositionError):
        ndgx.run_partitioned(cfg, _u0(cfg), 5)


def test_step_by_step_launch_sequence(monkeypatch):
    """NDGX_EAGER=1: the launch sequence blocks on several GPUs take (no CUDA
    graphs, cross-stream events only), here with every block on one device."""
    monkeypatch.setenv("NDGX_EAGER", "1")
    cfg = _cfg(2, (16, 16), 8, True)
    u0 = _u0(cfg)
    plan = ndgx.StepPlan(5, True)
    _, got, st, _, _ = _part(cfg, u0, 4, plan, ndgx.ARITH_FAST)
    monkeypatch.delenv("NDGX_EAGER")
    _, want, st_want = _single(cfg, u0, plan, ndgx.ARITH_FAST)
    assert np.array_equal(got, want) and st.dt_max == st_want.dt_max
    cfg.t_end = 0.01
    monkeypatch.setenv("NDGX_EAGER", "1")
    res = ndgx.run_partitioned(cfg, u0, 2)
    monkeypatch.delenv("NDGX_EAGER")
    want = ndgx.advance(cfg, u0)
    assert res.stats.steps == want.stats.steps and np.array_equal(res.state, want.state)
