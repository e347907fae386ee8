"""Multi-GPU block decomposition and face-halo exchange.

The GPU path (include/ndgx.h, ndgx_create_rank) is run_partitioned
(src/partition.cpp:186-333) with NCCL in place of the in-process Transport:
per RK stage every rank packs the stage-input planes of its split axes in the
layout [cross-section cell][var][face node] and posts, per axis,
    send(high plane -> nbr_high), recv(low halo <- nbr_low),
    send(low plane  -> nbr_low),  recv(high halo <- nbr_high).

CPU tests (gloo, world size 2) check the plan and execute exactly that
message schedule on planes packed by a numpy restatement of the device
layout; GPU tests run the real NCCL path on one B200 with every axis routed
through the transport (NCCL send/recv to self) and compare bit-for-bit with
the single-block solver.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import paper_2510_05254_b200 as ndgx


def _cfg(dim, cells, order, euler, rk=ndgx.RK4):
    mesh = ndgx.Mesh(dim, cells, order)
    model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if euler else ndgx.EquationModel.advection(dim, (1, 0, 0))
    return ndgx.SolverConfig(mesh, model, rk, 0.4, 1.0)


def _field(u_aos, cfg, cells):
    """Block AoS field -> array [c0][c1][c2][i][j][k][v] (unused axes of size 1)."""
    d, n = cfg.mesh.dim, cfg.mesh.order
    nodes = [n if a < d else 1 for a in range(3)]
    return u_aos.reshape(tuple(cells) + tuple(nodes) + (cfg.model.n_var(),))


def pack_plane(f, cfg, axis, side):
    """numpy restatement of pack_kernel (csrc/ndgx_device.cuh): the face plane
    [cross-section cell][var][face node] of a block field f (see _field)."""
    n = cfg.mesh.order
    dim = cfg.mesh.dim
    k = n - 1 if side else 0
    c = f.shape[axis] - 1 if side else 0
    # select the boundary cells and the boundary node along `axis`
    g = np.take(np.take(f, [c], axis=axis), [k], axis=3 + axis)
    g = np.squeeze(g, axis=(axis, 3 + axis))  # [ca][cb][na][nb][v] over the two other axes (ascending)
    # device order: cross-section cell with the lower other axis fastest,
    # face node with the lower other axis fastest, var in between
    ca, cb, na, nb, nv = g.shape
    g = g.transpose(1, 0, 4, 3, 2)  # [cb][ca][v][nb][na]
    if dim == 1:
        return g.reshape(-1)
    return g.reshape(cb * ca, nv, nb * na).reshape(-1)


# ------------------------------------------------------------------ CPU
@pytest.mark.parametrize("dim,cells,order,euler,ranks", [
    (2, (12, 10), 8, True, [1, 2, 3, 4, 6]),
    (3, (6, 4, 8), 4, True, [2, 4, 8]),
    (1, (64,), 4, False, [2, 4]),
])
def test_plan_tiles_the_mesh_and_is_symmetric(dim, cells, order, euler, ranks):
    cfg = _cfg(dim, cells, order, euler)
    for nr in ranks:
        plans = [ndgx.plan_rank(cfg, nr, r) for r in range(nr)]
        seen = np.zeros(tuple(cfg.mesh.cells), dtype=int)
        for r, pl in enumerate(plans):
            assert pl.rank == r and pl.nranks == nr
            sl = tuple(slice(pl.lo[a], pl.hi[a]) for a in range(3))
            seen[sl] += 1
            for a in range(3):
                assert bool(pl.split[a]) == (a < dim and pl.grid[a] > 1)
                lo_n, hi_n = plans[pl.nbr[a][0]], plans[pl.nbr[a][1]]
                assert hi_n.nbr[a][0] == r and lo_n.nbr[a][1] == r
                if pl.split[a]:  # both ends of every message agree on its size
                    assert lo_n.plane[a] == pl.plane[a] == hi_n.plane[a]
        assert (seen == 1).all()


@pytest.mark.parametrize("dim,cells,order", [(2, (12, 10), 8), (3, (6, 4, 8), 4)])
def test_block_initial_condition_is_the_global_slice(dim, cells, order):
    cfg = _cfg(dim, cells, order, True)
    g = _field(ndgx.init_euler_subsonic(cfg.mesh, cfg.model), cfg, cfg.mesh.cells)
    for r in range(4):
        pl = ndgx.plan_rank(cfg, 4, r)
        b = ndgx.init_block(cfg, pl.lo, pl.hi)
        want = g[tuple(slice(pl.lo[a], pl.hi[a]) for a in range(3))].reshape(-1)
        assert np.array_equal(b, want)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dim, cells, order = case
        cfg = _cfg(dim, cells, order, True)
        glob = _field(ndgx.init_euler_subsonic(cfg.mesh, cfg.model), cfg, cfg.mesh.cells)
        pl = ndgx.plan_rank(cfg, world, rank)
        mine = _field(ndgx.init_block(cfg, pl.lo, pl.hi), cfg, pl.cells())
        recv = {}
        for a in range(dim):
            if not pl.split[a]:
                continue
            n = int(pl.plane[a])
            bufs = [torch.empty(n, dtype=torch.float64) for _ in range(2)]
            # the C++ posting order (ndgx_solver.cu launch_exchange)
            ops = [dist.P2POp(dist.isend, torch.from_numpy(pack_plane(mine, cfg, a, 1)), pl.nbr[a][1]),
                   dist.P2POp(dist.irecv, bufs[0], pl.nbr[a][0]),
                   dist.P2POp(dist.isend, torch.from_numpy(pack_plane(mine, cfg, a, 0)), pl.nbr[a][0]),
                   dist.P2POp(dist.irecv, bufs[1], pl.nbr[a][1])]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            recv[a] = [b.numpy() for b in bufs]
        # each received halo is the neighbour cells' facing trace of the GLOBAL
        # field -- what the single-block kernel reads by periodic wrap
        ok = True
        for a, (lo_h, hi_h) in recv.items():
            for side, got in ((0, lo_h), (1, hi_h)):
                c = (pl.lo[a] - 1) % cfg.mesh.cells[a] if side == 0 else pl.hi[a] % cfg.mesh.cells[a]
                sl = [slice(pl.lo[b], pl.hi[b]) for b in range(3)]
                sl[a] = slice(c, c + 1)
                nb = glob[tuple(sl)]
                want = pack_plane(nb, cfg, a, 1 - side)  # its facing side
                ok = ok and np.array_equal(got, want)
        q.put((rank, ok, sorted(recv)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [(2, (12, 10), 8), (3, (4, 6, 8), 4)])
def test_gloo_two_rank_halo_exchange_matches_global_traces(case):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(axes for _, _, axes in res)  # some axis was actually exchanged


# ------------------------------------------------------------------ GPU
@pytest.fixture(scope="module")
def nccl_id():
    return ndgx.nccl_unique_id()


GPU_CASES = [
    ("2D Euler o8 RK4", (2, (12, 10), 8, True, ndgx.RK4)),
    ("3D Euler o4 RK6", (3, (4, 6, 5), 4, True, ndgx.RK6)),
    ("2D adv o3 RK3", (2, (9, 7), 3, False, ndgx.RK3)),
    ("1D adv o4 RK4", (1, (64,), 4, False, ndgx.RK4)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,case", GPU_CASES)
def test_nccl_self_exchange_bitwise_equals_single_block(name, case):
    dim, cells, order, euler, rk = case
    cfg = _cfg(dim, cells, order, euler, rk)
    u0 = ndgx.init_euler_subsonic(cfg.mesh, cfg.model) if euler else \
        ndgx.init_multisine(cfg.mesh, cfg.model, n_modes=5, seed=3)
    with ndgx.Solver(cfg) as s:
        s.upload(u0)
        r_want = s.rhs()
        st_want = s.advance(ndgx.StepPlan(7, True))
        want = s.download()
    with ndgx.Solver.for_rank(cfg, 1, 0, ndgx.nccl_unique_id(), force_exchange=True) as s:
        assert all(s.plan.split[a] for a in range(dim))
        s.upload(u0)
        r_got = s.rhs()
        st = s.advance(ndgx.StepPlan(7, True))
        got = s.download()
    assert np.array_equal(r_got, r_want), f"{name}: rhs through the transport differs"
    assert np.array_equal(got, want), f"{name}: state through the transport differs"
    assert (st.steps, st.dt_min, st.dt_max) == (st_want.steps, st_want.dt_min, st_want.dt_max)


@pytest.mark.gpu
def test_nccl_self_exchange_fast_mode_and_t_end(nccl_id):
    cfg = _cfg(2, (16, 12), 8, True)
    cfg.t_end = 0.02
    u0 = ndgx.init_euler_subsonic(cfg.mesh, cfg.model)
    res = []
    for rank_solver in (False, True):
        s = (ndgx.Solver.for_rank(cfg, 1, 0, nccl_id, arith=ndgx.ARITH_FAST, force_exchange=True)
             if rank_solver else ndgx.Solver(cfg, arith=ndgx.ARITH_FAST))
        with s:
            s.upload(u0)
            st = s.advance(ndgx.StepPlan(-1, False))
            res.append((s.download(), st))
    (a, sa), (b, sb) = res
    assert sa.steps == sb.steps and sa.dt_min == sb.dt_min
    assert np.array_equal(a, b)  # same kernels, same arithmetic, same halos


@pytest.mark.gpu
@pytest.mark.parametrize("plan", [ndgx.StepPlan(5, False), ndgx.StepPlan(-1, False)])
def test_rank_solver_errors_match_the_single_block(plan):
    """A PhysicsError through the transport path: same exception, same message,
    in fixed-step and t_end mode (the stop decision is all-reduced, so a rank
    never leaves collectives unmatched)."""
    cfg = _cfg(2, (12, 10), 8, True)
    cfg.t_end = 0.05
    u0 = ndgx.init_euler_subsonic(cfg.mesh, cfg.model)
    f = _field(u0.copy(), cfg, cfg.mesh.cells)
    f[3, 2, 0, 1, 5, 0, 0] = -0.5  # a negative density in cell (3, 2)
    bad = f.reshape(-1)
    msgs = []
    for ranked in (False, True):
        s = ndgx.Solver.for_rank(cfg, 1, 0, ndgx.nccl_unique_id(), force_exchange=True) if ranked else ndgx.Solver(cfg)
        with s:
            s.upload(bad)
            with pytest.raises(ndgx.PhysicsError) as ei:
                s.advance(plan)
            msgs.append(str(ei.value))
    assert msgs[0] == msgs[1]
