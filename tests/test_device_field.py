"""Initial conditions and diagnostics on the device.

init_multisine / init_euler_subsonic (src/grid.cpp:135-188), l2_error /
conserved_totals / l1_norm (src/grid.cpp:190-223) evaluated in HBM on the
solver's own layout.  The checker is the host restatement, which is the
reference bit for bit (tests/test_oracle.py): the device IC may differ only
through CUDA's sin (<= 2 ulp), the diagnostics only through the summation
order.  Tolerances: ICs 1e-14 relative to the field's max, diagnostics
1e-13 relative to the sum of |terms|.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2510_05254_b200 as ndgx

pytestmark = pytest.mark.gpu

CASES = [
    # (dim, cells, order, euler, length)
    (2, (24, 16), 8, True, (1.0, 1.0)),
    (2, (7, 5), 5, True, (2.0, 0.5)),
    (3, (6, 5, 4), 4, True, (1.0, 1.0, 1.0)),
    (1, (64,), 4, False, (1.0,)),
    (2, (12, 9), 3, False, (1.5, 1.0)),
    (3, (4, 3, 5), 6, False, (1.0, 2.0, 1.0)),
]
N_MODES, SEED = 7, 11


def _setup(dim, cells, order, euler, length):
    mesh = ndgx.Mesh(dim, cells, order, length)
    model = (ndgx.EquationModel.isothermal_euler(dim, 1.3) if euler
             else ndgx.EquationModel.advection(dim, (1.0, 0.5, 0.25)))
    cfg = ndgx.SolverConfig(mesh, model, ndgx.RK4, 0.4, 1.0)
    if euler:
        return cfg, ndgx.IC_EULER_SUBSONIC, None, ndgx.init_euler_subsonic(mesh, model)
    amps = ndgx.multisine_amplitudes(N_MODES, SEED)
    return cfg, ndgx.IC_MULTISINE, amps, ndgx.init_multisine(mesh, model, amplitudes=amps)


def _weights(cfg):
    """w of every node in the AoS order (for_each_node, src/grid.cpp:28-48)."""
    mesh = cfg.mesh
    _, w = ndgx.gauss_lobatto(mesh.order)
    jac = 1.0
    for a in range(mesh.dim):
        jac *= 0.5 * mesh.cell_size(a)
    wn = np.ones([mesh.order] * mesh.dim)
    for a in range(mesh.dim):
        shape = [1] * mesh.dim
        shape[a] = mesh.order
        wn = wn * np.asarray(w).reshape(shape)
    per_cell = (jac * wn).reshape(-1)
    return np.tile(np.repeat(per_cell, cfg.model.n_var()), mesh.cell_count())


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}D-o{c[2]}-{'euler' if c[3] else 'adv'}")
def test_device_ic_matches_host(case):
    cfg, ic, amps, host = _setup(*case)
    with ndgx.Solver(cfg, arith=ndgx.ARITH_FAST) as s:
        s.init_device(ic, amps)
        dev = s.download()
    scale = np.max(np.abs(host))
    assert np.max(np.abs(dev - host)) <= 1e-14 * scale


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}D-o{c[2]}-{'euler' if c[3] else 'adv'}")
def test_device_diagnostics_match_host(case):
    cfg, ic, amps, host = _setup(*case)
    mesh, model = cfg.mesh, cfg.model
    w = _weights(cfg)
    with ndgx.Solver(cfg, arith=ndgx.ARITH_FAST) as s:
        s.upload(host)
        s.advance(ndgx.StepPlan(3, False))
        u = s.download()
        tot = s.conserved_totals_device()
        want_tot = ndgx.conserved_totals(mesh, model, u)
        nv = model.n_var()
        absum = [np.sum(w[v::nv] * np.abs(u[v::nv])) for v in range(nv)]
        for v in range(nv):
            assert abs(tot[v] - want_tot[v]) <= 1e-13 * absum[v]
            l1 = s.l1_norm_device(v)
            assert abs(l1 - absum[v]) <= 1e-13 * absum[v]
            l2 = s.l2_error_ic_device(ic, amps, v)
            want = ndgx.l2_error(mesh, model, u, host, v)
            assert abs(l2 - want) <= 1e-13 * max(want, 1e-300) + 1e-15 * np.sqrt(np.sum(w[v::nv] * host[v::nv] ** 2))


def test_device_ic_on_partitioned_handle_equals_single_block():
    cfg, ic, amps, _ = _setup(2, (16, 12), 8, True, (1.0, 1.0))
    with ndgx.Solver(cfg, arith=ndgx.ARITH_FAST) as s:
        s.init_device(ic)
        single = s.download()
        tot1 = s.conserved_totals_device()
    with ndgx.Solver.partitioned(cfg, 4, arith=ndgx.ARITH_FAST) as s:
        s.init_device(ic)
        part = s.download()
        tot4 = s.conserved_totals_device()
        st = s.advance(ndgx.StepPlan(2, False))
    assert np.array_equal(part, single)
    assert np.allclose(tot4, tot1, rtol=1e-13, atol=1e-15)
    assert st.steps == 2


def test_device_ic_errors_match_the_reference():
    cfg, _, _, _ = _setup(2, (4, 4), 4, True, (1.0, 1.0))
    with ndgx.Solver(cfg) as s:
        with pytest.raises(ndgx.ConfigError, match="init_multisine applies to the advection scalar only"):
            s.init_device(ndgx.IC_MULTISINE, [1.0])
    cfg, _, _, _ = _setup(1, (8,), 4, False, (1.0,))
    with ndgx.Solver(cfg) as s:
        with pytest.raises(ndgx.ConfigError, match="init_euler_subsonic requires an isothermal Euler model"):
            s.init_device(ndgx.IC_EULER_SUBSONIC)
        with pytest.raises(ndgx.ConfigError, match="multisine: need at least one mode"):
            s.init_device(ndgx.IC_MULTISINE, [])
        with pytest.raises(ndgx.ConfigError, match="l1_norm: bad variable"):
            s.l1_norm_device(1)
