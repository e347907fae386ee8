"""Small runs of every stage-kernel body for compute-sanitizer (racecheck / synccheck / memcheck).

    compute-sanitizer --tool racecheck python scripts/sanitize_target.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_05254_b200 as ndgx  # noqa: E402

CASES = [
    # (name, dim, cells, order, euler, rk, arith, depth env)
    ("flagship 2D Euler o8 fast (DMMA, x-runs)", 2, (8, 6), 8, True, ndgx.RK4, ndgx.ARITH_FAST, None),
    ("2D advection o8 fast (DMMA, TMA ring)", 2, (8, 6), 8, False, ndgx.RK4, ndgx.ARITH_FAST, None),
    ("3D Euler o4 RK6 fast (DMMA, z-runs)", 3, (4, 3, 5), 4, True, ndgx.RK6, ndgx.ARITH_FAST, None),
    ("2D Euler o8 exact (generic, ring forced)", 2, (6, 5), 8, True, ndgx.RK4, ndgx.ARITH_EXACT, "3"),
    ("2D Euler o4 fast (8 lanes per element)", 2, (9, 7), 4, True, ndgx.RK3, ndgx.ARITH_FAST, None),
    ("1D advection o3 exact (4 lanes per element, ring)", 1, (33,), 3, False, ndgx.RK4, ndgx.ARITH_EXACT, None),
    ("3D advection o2 (8 lanes per element)", 3, (3, 4, 5), 2, False, ndgx.RK4, ndgx.ARITH_FAST, None),
    ("3D Euler o4 RK6 fast, 16 z planes (line body, z-runs of 8)", 3, (3, 2, 16), 4, True, ndgx.RK6,
     ndgx.ARITH_FAST, None),
    ("2D Euler o8 exact (line-task volume)", 2, (5, 4), 8, True, ndgx.RK4, ndgx.ARITH_EXACT, None),
    ("2D Euler o6 fast (flagship body zero-padded to 8 x 8, x-runs)", 2, (7, 5), 6, True, ndgx.RK4, ndgx.ARITH_FAST,
     None),
    ("2D Euler o7 fast (flagship body zero-padded, odd N)", 2, (5, 6), 7, True, ndgx.RK6, ndgx.ARITH_FAST, None),
    ("2D advection o7 fast (flagship body zero-padded)", 2, (4, 5), 7, False, ndgx.RK4, ndgx.ARITH_FAST, None),
    ("2D Euler o6 exact (whole-line volume, 8 lanes per element)", 2, (7, 5), 6, True, ndgx.RK4, ndgx.ARITH_EXACT,
     None),
    ("2D advection o7 exact (whole-line volume)", 2, (4, 3), 7, False, ndgx.RK3, ndgx.ARITH_EXACT, None),
]
for name, dim, cells, order, euler, rk, arith, depth in CASES:
    if depth is None:
        os.environ.pop("NDGX_DEPTH", None)
    else:
        os.environ["NDGX_DEPTH"] = depth
    mesh = ndgx.Mesh(dim, cells, order)
    model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if euler else ndgx.EquationModel.advection(dim, (1, .5, .2))
    cfg = ndgx.SolverConfig(mesh, model, rk, 0.4, 1.0)
    with ndgx.Solver(cfg, arith=arith) as s:
        s.init_device(ndgx.IC_EULER_SUBSONIC if euler else ndgx.IC_MULTISINE,
                      None if euler else ndgx.multisine_amplitudes(3, 5))
        s.advance(ndgx.StepPlan(2, False))
        s.rhs()
    with ndgx.Solver.partitioned(cfg, 2, arith=arith) as s:  # pack kernels and split stages
        s.init_device(ndgx.IC_EULER_SUBSONIC if euler else ndgx.IC_MULTISINE,
                      None if euler else ndgx.multisine_amplitudes(3, 5))
        s.advance(ndgx.StepPlan(2, False))
    print("ok", name, flush=True)
