"""Checkpoint / restart in the reference's field-dump format.

dump_field / load_field (src/field_io.cpp:18-72, include/ndg/field_io.hpp):
"ndgfield 1", one "key values" header line each for dim, cells, order,
nvar and length, a "data" line, then the raw little-endian doubles in
FieldShape::index order.  The reference's own test is "field dump
round-trips bit for bit" (proj/tests/test_grid.cpp:236-255).
"""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

import paper_2510_05254_b200 as ndgx

CASES = [
    # (dim, cells, order, euler, length)
    (2, (3, 2), 3, True, (2.0, 1.0)),           # the reference's own case
    (2, (5, 4), 8, True, (0.3, 1.0 / 3.0)),     # %g-formatted lengths
    (3, (2, 3, 2), 4, True, (1.0, 12345.678, 2.5e-7)),
    (1, (16,), 4, False, (1.0,)),
]


def _field(dim, cells, order, euler, length):
    mesh = ndgx.Mesh(dim, cells, order, length)
    model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if euler else ndgx.EquationModel.advection(dim, (1,))
    u = ndgx.init_euler_subsonic(mesh, model) if euler else ndgx.init_multisine(mesh, model, n_modes=3, seed=7)
    return mesh, model, u


REF_DUMP = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "ref_dump")


@pytest.mark.parametrize("case", CASES)
def test_host_dump_is_byte_identical_to_the_reference(tmp_path, case):
    if not os.path.exists(REF_DUMP):
        pytest.skip("tests/cpp/_build/ref_dump not built (needs /root/reference at build time)")
    dim, cells, order, euler, length = case
    mesh, model, u = _field(*case)
    ours, ref, raw = tmp_path / "ours.ndgf", tmp_path / "ref.ndgf", tmp_path / "u.f64"
    ndgx.dump_field(str(ours), mesh, u)
    u.astype("<f8").tofile(raw)
    c3 = list(mesh.cells)
    l3 = list(mesh.length)
    subprocess.run([REF_DUMP, str(dim), *map(str, c3), str(order), "1" if euler else "0",
                    *(repr(x) for x in l3), str(raw), str(ref)], check=True)
    assert ours.read_bytes() == ref.read_bytes()


@pytest.mark.parametrize("case", CASES)
def test_load_round_trips_bit_for_bit(tmp_path, case):
    mesh, model, u = _field(*case)
    path = tmp_path / "f.ndgf"
    ndgx.dump_field(str(path), mesh, u)
    dim, cells, order, nvar, length, f = ndgx.load_field(str(path))
    assert (dim, cells, order, nvar) == (mesh.dim, tuple(mesh.cells[:mesh.dim]), mesh.order, model.n_var())
    assert np.array_equal(f, u)
    assert length[0] == float(f"{mesh.length[0]:g}")


def test_load_rejects_broken_files(tmp_path):
    mesh, model, u = _field(*CASES[0])
    good = tmp_path / "good.ndgf"
    ndgx.dump_field(str(good), mesh, u)
    raw = good.read_bytes()
    with pytest.raises(FileNotFoundError):
        ndgx.load_field(str(tmp_path / "does_not_exist.ndgf"))
    bad = tmp_path / "bad.ndgf"
    bad.write_bytes(b"ndgfield 2\n" + raw.split(b"\n", 1)[1])
    with pytest.raises(RuntimeError, match="not an ndgfield dump"):
        ndgx.load_field(str(bad))
    bad.write_bytes(raw[: len(raw) - 8])
    with pytest.raises(RuntimeError, match="truncated payload"):
        ndgx.load_field(str(bad))
    bad.write_bytes(raw.replace(b"order", b"degree"))
    with pytest.raises(RuntimeError, match="unknown header key"):
        ndgx.load_field(str(bad))


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES[:3])
def test_device_dump_matches_host_dump(tmp_path, case):
    mesh, model, u = _field(*case)
    with ndgx.Solver(ndgx.SolverConfig(mesh, model)) as s:
        s.upload(u)
        s.advance(ndgx.StepPlan(3))
        got = s.download()
        s.dump_field(str(tmp_path / "dev.ndgf"))
    ndgx.dump_field(str(tmp_path / "host.ndgf"), mesh, got)
    assert (tmp_path / "dev.ndgf").read_bytes() == (tmp_path / "host.ndgf").read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("arith", [ndgx.ARITH_EXACT, ndgx.ARITH_FAST])
def test_checkpoint_restart_is_bit_identical(tmp_path, arith):
    mesh, model, u = _field(2, (12, 10), 8, True, (1.0, 1.0))
    cfg = ndgx.SolverConfig(mesh, model)
    with ndgx.Solver(cfg, arith=arith) as s:
        s.upload(u)
        s.advance(ndgx.StepPlan(10))
        want = s.download()
    path = str(tmp_path / "ckpt.ndgf")
    with ndgx.Solver(cfg, arith=arith) as s:
        s.upload(u)
        s.advance(ndgx.StepPlan(6))
        s.dump_field(path)
    with ndgx.Solver(cfg, arith=arith) as s:
        s.load_field(path)
        s.advance(ndgx.StepPlan(4))
        got = s.download()
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_load_checks_the_mesh(tmp_path):
    mesh, model, u = _field(*CASES[0])
    path = str(tmp_path / "f.ndgf")
    ndgx.dump_field(path, mesh, u)
    other = ndgx.Mesh(2, (4, 2), 3, (2.0, 1.0))
    with ndgx.Solver(ndgx.SolverConfig(other, model)) as s:
        with pytest.raises(ndgx.ConfigError, match="does not match"):
            s.load_field(path)
