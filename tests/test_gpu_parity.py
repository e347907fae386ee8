"""GPU parity: the sm_100a path (through the C ABI) against the oracle and the
reference's golden vectors.

Bar (SURVEY.md §8c / north_star):
* NDGX_ARITH_EXACT: bit-identical states, RHS and step statistics
  (FNV-1a digests equal to the reference's);
* NDGX_ARITH_FAST (FMA-contracted): per-variable relative GL-L2 <= 1e-12
  after the fixed steps (tolerance written below as REL_L2_TOL);
* integer work (layout permutation, decomposition): exact.
"""
import os

import numpy as np
import pytest

from oracle_lib import ADVECTION, EULER, RK3, RK4, RK6, Problem, fnv1a64, rel_l2
from test_oracle import APPENDIX, SMALL, initial_from, problem_from

import paper_2510_05254_b200 as ndgx

pytestmark = pytest.mark.gpu

REL_L2_TOL = 1e-12


def config_of(p: Problem) -> ndgx.SolverConfig:
    mesh = ndgx.Mesh(p.dim, p.cells3[:p.dim], p.order, p.length)
    if p.kind == EULER:
        model = ndgx.EquationModel.isothermal_euler(p.dim, p.sound_speed)
    else:
        model = ndgx.EquationModel.advection(p.dim, p.velocity)
    return ndgx.SolverConfig(mesh, model, p.rk, p.cfl, p.t_end)


def test_device_is_b200():
    import torch
    assert torch.cuda.is_available()
    assert torch.cuda.get_device_capability(0) == (10, 0)


@pytest.mark.parametrize("name", SMALL + APPENDIX)
def test_exact_mode_bitwise_equals_reference(port, golden, golden_states, name):
    case = golden["cases"][name]
    p = problem_from(case["problem"])
    u0 = golden_states.get(name + "/init")
    if u0 is None:
        u0 = initial_from(port, p, case["ic"])
    assert fnv1a64(u0) == case["digest_init"]
    with ndgx.Solver(config_of(p), arith=ndgx.ARITH_EXACT) as s:
        s.upload(u0)
        assert np.array_equal(s.download(), u0)  # AoS <-> device layout round trip
        r0 = s.rhs()
        assert fnv1a64(r0) == case["digest_rhs0"], f"rhs max |diff| {np.abs(r0 - port.rhs(p, u0)).max()}"
        st = s.advance(ndgx.StepPlan(case["fixed_steps"], False))
        uf = s.download()
    if fnv1a64(uf) != case["digest_final"]:
        want, _ = port.advance(p, u0, case["fixed_steps"])
        pytest.fail(f"final state differs: rel L2 {rel_l2(port, p, uf, want)}")
    assert st.steps == case["steps"] and st.dt_min == case["dt_min"] and st.dt_max == case["dt_max"]


@pytest.mark.parametrize("name", SMALL + APPENDIX)
def test_fast_mode_within_tolerance(port, golden, golden_states, name):
    case = golden["cases"][name]
    p = problem_from(case["problem"])
    u0 = initial_from(port, p, case["ic"])
    want = golden_states.get(name + "/final")
    if want is None:
        want, _ = port.advance(p, u0, case["fixed_steps"])
    with ndgx.Solver(config_of(p), arith=ndgx.ARITH_FAST) as s:
        s.upload(u0)
        r0 = s.rhs()
        st = s.advance(ndgx.StepPlan(case["fixed_steps"], False))
        uf = s.download()
    r_want = port.rhs(p, u0)
    assert max(rel_l2(port, p, r0, r_want)) <= REL_L2_TOL
    errs = rel_l2(port, p, uf, want)
    assert max(errs) <= REL_L2_TOL, errs
    assert st.steps == case["steps"]


@pytest.mark.parametrize("name", ["tend_adv1d_o4_10", "tend_adv2d_o3_6", "tend_short_adv1d",
                                  "tend_euler2d_o4_6", "tend_zero_wavespeed"])
def test_t_end_landing_bitwise(golden, golden_states, name):
    case = golden["t_end"][name]
    p = problem_from(case["problem"])
    with ndgx.Solver(config_of(p)) as s:
        s.upload(golden_states[name + "/init"])
        st = s.advance(ndgx.StepPlan(-1, False))
        uf = s.download()
    assert st.steps == case["steps"]
    assert st.dt_max == case["dt_max"] and st.dt_min == case["dt_min"]
    assert fnv1a64(uf) == case["digest_final"]


def test_warmup_does_not_change_the_result(golden, golden_states):
    case = golden["cases"]["euler2d_o3_rk4_8"]
    p = problem_from(case["problem"])
    with ndgx.Solver(config_of(p)) as s:
        s.upload(golden_states["euler2d_o3_rk4_8/init"])
        st = s.advance(ndgx.StepPlan(case["fixed_steps"], True))
        assert fnv1a64(s.download()) == case["digest_final"] and st.steps == case["steps"]


def test_error_semantics_match_reference(golden, golden_states):
    g = golden["errors"]
    p = Problem(2, (4, 4), 3, EULER, RK4)
    with ndgx.Solver(config_of(p)) as s:
        s.upload(golden_states["err_rho/init"])
        with pytest.raises(ndgx.PhysicsError) as e:
            s.rhs()
        assert str(e.value) == g["negative_density_rhs"]["message"]
        with pytest.raises(ndgx.PhysicsError) as e:
            s.advance(ndgx.StepPlan(4, False))
        assert str(e.value) == g["negative_density_advance"]["message"]
    p = Problem(1, (8,), 3, ADVECTION, RK4)
    with ndgx.Solver(config_of(p)) as s:
        s.upload(golden_states["err_nan/init"])
        with pytest.raises(ndgx.InstabilityError) as e:
            s.advance(ndgx.StepPlan(-1, False))
        assert e.value.step == 1 and str(e.value) == g["nan_state"]["message"]
    p = Problem(1, (8,), 3, ADVECTION, RK4, velocity=(0.0, 0.0, 0.0))
    with ndgx.Solver(config_of(p)) as s:
        s.upload(np.ones(p.size))
        with pytest.raises(ndgx.ConfigError) as e:
            s.advance(ndgx.StepPlan(3, False))
        assert str(e.value) == g["zero_wavespeed_fixed"]["message"]


def test_negative_density_mid_run_names_the_cell(port):
    """A density that turns negative inside a stage is reported like the
    reference's apply() (solver.cpp:258-261) with the offending cell."""
    p = Problem(2, (6, 5), 4, EULER, RK4)
    u = port.init_euler(p)
    u[0::3] *= 1e-3  # tiny density -> large velocities -> failure within a few steps
    u[1::3] += 0.5
    try:
        port.advance(p, u, 50)
        pytest.skip("state did not fail in the oracle")
    except Exception as e:  # noqa: BLE001
        want = e.message
    with ndgx.Solver(config_of(p)) as s:
        s.upload(u)
        with pytest.raises((ndgx.PhysicsError, ndgx.InstabilityError)) as got:
            s.advance(ndgx.StepPlan(50, False))
    assert str(got.value) == want


def test_mid_size_euler_o8_bitwise(port):
    """2D isothermal Euler o8 RK4 at 96^2 cells (1.77e6 DOF), 10 steps."""
    p = Problem(2, (96, 96), 8, EULER, RK4)
    u0 = port.init_euler(p)
    want, st_w = port.advance(p, u0, 10)
    with ndgx.Solver(config_of(p)) as s:
        s.upload(u0)
        st = s.advance(ndgx.StepPlan(10, True))
        got = s.download()
    assert np.array_equal(got, want)
    assert st.dt_min == st_w.dt_min and st.dt_max == st_w.dt_max


def test_rhs_of_constant_state_vanishes():
    """test_solver.cpp:119-157."""
    cfg = ndgx.SolverConfig(ndgx.Mesh(2, (16, 16), 8), ndgx.EquationModel.isothermal_euler(2, 1.0))
    u = np.zeros(16 * 16 * 64 * 3)
    u[0::3], u[1::3], u[2::3] = 1.0, 0.3, -0.2
    with ndgx.Solver(cfg) as s:
        s.upload(u)
        assert np.abs(s.rhs()).max() <= 1e-12


def test_conservation_and_determinism_large(port):
    """Conserved totals drift <= 1e-12 (test_solver.cpp:396-409) and bitwise
    determinism (:367-378) on 2D Euler o8 at 192^2 cells, 20 steps."""
    p = Problem(2, (192, 192), 8, EULER, RK4)
    mesh = ndgx.Mesh(2, (192, 192), 8)
    u0 = ndgx.init_euler_subsonic(mesh, ndgx.EquationModel.isothermal_euler(2, 1.0))
    outs = []
    for _ in range(2):
        with ndgx.Solver(config_of(p)) as s:
            s.upload(u0)
            s.advance(ndgx.StepPlan(20, False))
            outs.append(s.download())
    assert np.array_equal(outs[0], outs[1])
    import ctypes as C
    t0, t1 = (np.zeros(3), np.zeros(3))
    c = p.ndgo()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    port.lib.ndgo_conserved_totals(C.byref(c), dp(u0), dp(t0))
    port.lib.ndgo_conserved_totals(C.byref(c), dp(outs[0]), dp(t1))
    for v in range(3):
        scale = max(port.lib.ndgo_l1_norm(C.byref(c), dp(u0), v), 1e-3)
        assert abs(t1[v] - t0[v]) / scale <= 1e-12


def test_advection_linearity():
    """test_solver.cpp:347-365."""
    mesh = ndgx.Mesh(2, (12, 9), 5)
    model = ndgx.EquationModel.advection(2, (1.0, 0.5, 0.0))
    cfg = ndgx.SolverConfig(mesh, model, ndgx.RK4, 0.4, 0.1)
    a = ndgx.init_multisine(mesh, model, n_modes=3, seed=100)
    b = ndgx.init_multisine(mesh, model, n_modes=3, seed=200)
    ra = ndgx.advance(cfg, a).state
    rb = ndgx.advance(cfg, b).state
    rs = ndgx.advance(cfg, a + b).state
    assert np.abs(rs - (ra + rb)).max() <= 1e-12


def test_convergence_order_on_gpu():
    """2D advection converges at the scheme order (test_solver.cpp:333-345),
    extended to finer grids than the CPU test runs."""
    errs = []
    for cells in (8, 16, 32):
        mesh = ndgx.Mesh(2, (cells, cells), 4)
        model = ndgx.EquationModel.advection(2, (1.0, 0.0, 0.0))
        f = ndgx.init_multisine(mesh, model, n_modes=2, seed=21)
        r = ndgx.advance(ndgx.SolverConfig(mesh, model, ndgx.RK6, 0.4, 1.0), f)
        from oracle_lib import Oracle
        errs.append(Oracle("port").l2_error(Problem(2, (cells, cells), 4, ADVECTION, RK6), r.state, f, 0))
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert min(rates) > 3.5, rates


def test_full_size_c3_rhs_bitwise_and_step_properties(port):
    """BASELINE config C3 (2D isothermal Euler o8, 768^2 cells, 1.13e8 DOF):
    RHS bit-identical to the oracle at full size; 2 steps exact == fast to
    1e-12 and conserved to 1e-12."""
    p = Problem(2, (768, 768), 8, EULER, RK4)
    mesh = ndgx.Mesh(2, (768, 768), 8)
    u0 = ndgx.init_euler_subsonic(mesh, ndgx.EquationModel.isothermal_euler(2, 1.0))
    with ndgx.Solver(config_of(p), arith=ndgx.ARITH_EXACT) as s:
        s.upload(u0)
        r = s.rhs()
        s.advance(ndgx.StepPlan(2, False))
        ue = s.download()
    assert np.array_equal(r, port.rhs(p, u0))
    with ndgx.Solver(config_of(p), arith=ndgx.ARITH_FAST) as s:
        s.upload(u0)
        s.advance(ndgx.StepPlan(2, False))
        uf = s.download()
    d = ue - uf
    for v in range(3):
        assert np.sqrt((d[v::3] ** 2).sum() / (ue[v::3] ** 2).sum()) <= REL_L2_TOL


# Every (dim, order, equation) kernel instance the registry compiles, on a tiny
# mesh against the oracle port: exact bitwise, fast within REL_L2_TOL.  This
# covers the bodies and lane groupings the golden cases do not name (2D o6,
# 1D o3/o5-o7, 3D o5-o8, the 3D line body under RK3/RK4 ...).
SHAPES = ([(1, o, ADVECTION) for o in range(2, 9)] + [(2, o, k) for o in range(2, 9) for k in (ADVECTION, EULER)] +
          [(3, o, k) for o in range(2, 9) for k in (ADVECTION, EULER)])
CELLS = {1: (9,), 2: (5, 4), 3: (3, 2, 3)}


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[0]}D-o{s[1]}-{'euler' if s[2] == EULER else 'adv'}")
def test_every_shape_matches_port(port, shape):
    dim, order, kind = shape
    rk = (RK3, RK4, RK6)[order % 3]
    p = Problem(dim, CELLS[dim], order, kind, rk, velocity=(1.0, -0.5, 0.25), sound_speed=1.0)
    cfg = config_of(p)
    if kind == EULER:
        u0 = ndgx.init_euler_subsonic(cfg.mesh, cfg.model)
    else:
        u0 = ndgx.init_multisine(cfg.mesh, cfg.model, n_modes=3, seed=5)
    steps = 3
    want, want_st = port.advance(p, u0, steps)
    r_want = port.rhs(p, u0)
    for arith in (ndgx.ARITH_EXACT, ndgx.ARITH_FAST):
        with ndgx.Solver(cfg, arith=arith) as s:
            s.upload(u0)
            r0 = s.rhs()
            st = s.advance(ndgx.StepPlan(steps, False))
            uf = s.download()
        if arith == ndgx.ARITH_EXACT:
            assert np.array_equal(r0, r_want) and np.array_equal(uf, want)
            assert st.dt_min == want_st.dt_min and st.dt_max == want_st.dt_max
        else:
            assert max(rel_l2(port, p, r0, r_want)) <= REL_L2_TOL
            assert max(rel_l2(port, p, uf, want)) <= REL_L2_TOL


def _ref_workers():
    return max(1, min(16, os.cpu_count() or 1))


def test_full_size_c3_five_steps_against_the_reference(reference):
    """C3 at full size (768^2 cells, 1.13e8 DOF), 5 CFL steps against the
    reference itself (its run_partitioned over the host's threads, whose
    states equal its serial advance): exact bitwise, fast within REL_L2_TOL."""
    p = Problem(2, (768, 768), 8, EULER, RK4)
    mesh = ndgx.Mesh(2, (768, 768), 8)
    u0 = ndgx.init_euler_subsonic(mesh, ndgx.EquationModel.isothermal_euler(2, 1.0))
    want, st_w = reference.run_partitioned(p, u0, _ref_workers(), 5)
    for arith in (ndgx.ARITH_EXACT, ndgx.ARITH_FAST):
        with ndgx.Solver(config_of(p), arith=arith) as s:
            s.upload(u0)
            st = s.advance(ndgx.StepPlan(5, False))
            got = s.download()
        if arith == ndgx.ARITH_EXACT:
            assert np.array_equal(got, want) and st.dt_min == st_w.dt_min and st.dt_max == st_w.dt_max
        else:
            d = got - want
            for v in range(3):
                assert np.sqrt((d[v::3] ** 2).sum() / (want[v::3] ** 2).sum()) <= REL_L2_TOL


@pytest.mark.parametrize("n,steps", [(64, 5), (128, 3)], ids=["64cubed", "128cubed_full_size"])
def test_3d_euler_rk6_against_the_reference(reference, n, steps):
    """The C4 shape (3D isothermal Euler o4 RK6) at 64^3 cells (6.7e7 DOF, 5
    steps) and at the benchmark size 128^3 (5.4e8 DOF, 3 steps) against the
    reference: exact bitwise, fast within REL_L2_TOL (the line body, z-runs)."""
    p = Problem(3, (n, n, n), 4, EULER, RK6)
    cfg = config_of(p)
    u0 = ndgx.init_euler_subsonic(cfg.mesh, cfg.model)
    want, st_w = reference.run_partitioned(p, u0, _ref_workers(), steps)
    for arith in (ndgx.ARITH_EXACT, ndgx.ARITH_FAST):
        with ndgx.Solver(cfg, arith=arith) as s:
            s.upload(u0)
            st = s.advance(ndgx.StepPlan(steps, False))
            got = s.download()
        if arith == ndgx.ARITH_EXACT:
            assert np.array_equal(got, want) and st.dt_max == st_w.dt_max
        else:
            d = got - want
            for v in range(4):
                den = (want[v::4] ** 2).sum()
                assert np.sqrt((d[v::4] ** 2).sum() / den) <= REL_L2_TOL if den > 0 else np.abs(d[v::4]).max() <= 1e-13


def test_full_size_c4_fast_equals_exact_and_conserves():
    """C4 at the benchmark size (128^3 cells, 5.4e8 DOF), 3 steps: the fast
    mode within REL_L2_TOL of the bit-identical mode, totals conserved."""
    cfg = ndgx.SolverConfig(ndgx.Mesh(3, (128, 128, 128), 4), ndgx.EquationModel.isothermal_euler(3, 1.0), ndgx.RK6)
    out = {}
    for arith in (ndgx.ARITH_EXACT, ndgx.ARITH_FAST):
        with ndgx.Solver(cfg, arith=arith) as s:
            s.init_device(ndgx.IC_EULER_SUBSONIC)
            t0 = s.conserved_totals_device()
            s.advance(ndgx.StepPlan(3, False))
            out[arith] = (s.download(), s.conserved_totals_device(), t0)
    ue, uf = out[ndgx.ARITH_EXACT][0], out[ndgx.ARITH_FAST][0]
    for v in range(4):
        den = (ue[v::4] ** 2).sum()
        d = np.sqrt(((ue[v::4] - uf[v::4]) ** 2).sum() / den) if den > 0 else np.abs(uf[v::4]).max()
        assert d <= REL_L2_TOL
    tot, t0 = out[ndgx.ARITH_FAST][1], out[ndgx.ARITH_FAST][2]
    assert abs(tot[0] - t0[0]) <= 1e-12 * abs(t0[0])


@pytest.mark.parametrize("dim,cells,order", [(3, (4, 3, 5), 4), (2, (6, 5), 8), (2, (7, 5), 4), (3, (3, 4, 2), 2),
                                             (2, (5, 6), 7), (2, (6, 4), 6)],
                         ids=["3D-o4-lines", "2D-o8-flagship", "2D-o4-groups", "3D-o2-groups", "2D-o7-padded",
                              "2D-o6-padded"])
@pytest.mark.parametrize("arith", [ndgx.ARITH_EXACT, ndgx.ARITH_FAST], ids=["exact", "fast"])
def test_operator_physics_error_names_the_cell_in_every_body(port, dim, cells, order, arith):
    """A non-positive density at one node: serial_rhs's PhysicsError
    (solver.cpp:258-261) names the same cell and value as the reference's,
    from every stage-kernel body, in both arithmetic modes."""
    p = Problem(dim, cells, order, EULER, RK4)
    cfg = config_of(p)
    u = ndgx.init_euler_subsonic(cfg.mesh, cfg.model)
    nv = dim + 1
    bad = (p.size // nv) // 2 + 1  # a node inside the mesh
    u[bad * nv] = -0.5
    with pytest.raises(Exception) as want:
        port.rhs(p, u)
    with ndgx.Solver(cfg, arith=arith) as s:
        s.upload(u)
        with pytest.raises(ndgx.PhysicsError) as got:
            s.rhs()
    assert str(got.value) == want.value.message


@pytest.mark.parametrize("dim,cells,order,kind", [
    (2, (1, 3), 8, EULER), (2, (2, 1), 8, EULER), (2, (1, 1), 8, ADVECTION), (2, (3, 1), 4, EULER),
    (3, (1, 1, 5), 4, EULER), (3, (2, 1, 1), 4, EULER), (3, (1, 2, 1), 4, ADVECTION), (1, (1,), 5, ADVECTION),
    (2, (1, 3), 7, EULER), (2, (2, 1), 6, ADVECTION), (2, (1, 1), 5, EULER),
], ids=lambda x: str(x).replace(" ", ""))
def test_degenerate_meshes_match_port(port, dim, cells, order, kind):
    """One-cell axes: the element is its own periodic neighbour (and runs,
    lane groups and z-runs degenerate to length 1); exact bitwise, fast
    within REL_L2_TOL."""
    p = Problem(dim, cells, order, kind, RK4 if dim < 3 else RK6, velocity=(1.0, 0.5, -0.25))
    cfg = config_of(p)
    u0 = (ndgx.init_euler_subsonic(cfg.mesh, cfg.model) if kind == EULER
          else ndgx.init_multisine(cfg.mesh, cfg.model, n_modes=2, seed=9))
    want, _ = port.advance(p, u0, 3)
    for arith in (ndgx.ARITH_EXACT, ndgx.ARITH_FAST):
        with ndgx.Solver(cfg, arith=arith) as s:
            s.upload(u0)
            s.advance(ndgx.StepPlan(3, False))
            got = s.download()
        if arith == ndgx.ARITH_EXACT:
            assert np.array_equal(got, want)
        else:
            assert max(rel_l2(port, p, got, want)) <= REL_L2_TOL
