"""CPU tests of the product's boundary: libndgx.so loads, exports every symbol
include/ndgx.h declares, and its host-side setup (basis, ICs, decomposition)
is bit-identical to the oracle.  No GPU compute here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle_lib import ADVECTION, EULER, Problem

import paper_2510_05254_b200 as ndgx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ndgx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ndgx_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ndgx.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert ndgx.version().endswith("sm_100a")


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", ndgx.ndgx.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_create_without_gpu_fails_loudly():
    """No CPU fallback: without a B200 the handle cannot be created."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    mesh = ndgx.Mesh(2, (4, 4), 3)
    cfg = ndgx.SolverConfig(mesh, ndgx.EquationModel.isothermal_euler(2, 1.0))
    with pytest.raises(ndgx.CudaError):
        ndgx.Solver(cfg)


def test_config_errors_before_device():
    mesh = ndgx.Mesh(2, (4, 4), 3)
    model = ndgx.EquationModel.isothermal_euler(2, 1.0)
    with pytest.raises(ndgx.ConfigError):
        ndgx.validate(ndgx.SolverConfig(mesh, model, ndgx.RK4, 0.0, 1.0))
    with pytest.raises(ndgx.ConfigError):
        ndgx.validate(ndgx.SolverConfig(mesh, model, ndgx.RK4, 1.5, 1.0))
    with pytest.raises(ndgx.ConfigError):
        ndgx.validate(ndgx.SolverConfig(mesh, model, ndgx.RK4, 0.4, 0.0))
    with pytest.raises(ndgx.ConfigError):
        ndgx.validate(ndgx.SolverConfig(ndgx.Mesh(1, (8,), 3), model))
    with pytest.raises(ndgx.ConfigError):
        ndgx.EquationModel.isothermal_euler(1, 1.0)
    with pytest.raises(ndgx.ConfigError):
        ndgx.rk_from_name("rk5")
    with pytest.raises(ndgx.ConfigError):
        ndgx.Mesh(2, (0, 4), 3)


@pytest.mark.parametrize("order", range(2, 17))
def test_basis_bit_identical_to_oracle(port, order):
    nodes, w = ndgx.gauss_lobatto(order)
    d = ndgx.differentiation_matrix(order, nodes)
    on, ow, od = port.basis(order)
    assert np.array_equal(nodes, on) and np.array_equal(w, ow) and np.array_equal(d, od)


@pytest.mark.parametrize("dim,cells,order,kind", [(1, (16,), 4, ADVECTION), (2, (5, 7), 8, ADVECTION),
                                                  (3, (3, 4, 2), 3, ADVECTION), (2, (6, 5), 7, EULER),
                                                  (3, (4, 3, 5), 4, EULER), (2, (200, 130), 3, EULER)])
def test_initial_conditions_bit_identical_to_oracle(port, dim, cells, order, kind):
    p = Problem(dim, cells, order, kind)
    mesh = ndgx.Mesh(dim, cells, order)
    if kind == EULER:
        got = ndgx.init_euler_subsonic(mesh, ndgx.EquationModel.isothermal_euler(dim, 1.0))
        want = port.init_euler(p)
    else:
        got = ndgx.init_multisine(mesh, ndgx.EquationModel.advection(dim, (1, 0, 0)), n_modes=5, seed=3)
        want = port.init_multisine(p, n_modes=5, seed=3)
    assert np.array_equal(got, want)


def test_amplitudes_splitmix_kats():
    """test_grid.cpp:77-91."""
    a = ndgx.multisine_amplitudes(3, 42)
    assert a.tolist() == [0.7415648787718233, 0.1599103928769201, 0.27860113025513866]


def test_decompose_matches_reference_kats(golden):
    for d in golden["decompose"]:
        mesh = ndgx.Mesh(d["dim"], tuple(d["cells"]), 2)
        dec = ndgx.decompose(mesh, d["workers"])
        assert list(dec.grid) == d["grid"]
        for w, b in enumerate(dec.blocks):
            assert list(b.lo) == d["lo"][w] and list(b.hi) == d["hi"][w]
            assert [list(x) for x in b.neighbor] == d["nbr"][w]
    with pytest.raises(ndgx.DecompositionError) as e:
        ndgx.decompose(ndgx.Mesh(2, (3, 2), 3), 7)
    assert "factorization" in str(e.value)
    with pytest.raises(ndgx.DecompositionError):
        ndgx.decompose(ndgx.Mesh(1, (4,), 3), 0)


def test_decompose_property_tiling_balance_symmetry():
    """test_partition.cpp:76-125: exact tiling, balance within one cell, symmetric wrap."""
    rng = np.random.default_rng(31)
    for _ in range(120):
        dim = int(rng.integers(1, 4))
        cells = [1, 1, 1]
        for a in range(dim):
            cells[a] = int(rng.integers(1, 14))
        workers = int(rng.integers(1, 13))
        try:
            dec = ndgx.decompose(ndgx.Mesh(dim, tuple(cells[:dim]), 2), workers)
        except ndgx.DecompositionError:
            continue
        cov = np.zeros(cells, dtype=int)
        for b in dec.blocks:
            cov[b.lo[0]:b.hi[0], b.lo[1]:b.hi[1], b.lo[2]:b.hi[2]] += 1
        assert (cov == 1).all()
        for a in range(3):
            ext = [b.hi[a] - b.lo[a] for b in dec.blocks]
            assert max(ext) - min(ext) <= 1
        for w, b in enumerate(dec.blocks):
            for a in range(3):
                assert dec.blocks[b.neighbor[a][1]].neighbor[a][0] == w
                assert dec.blocks[b.neighbor[a][0]].neighbor[a][1] == w
