import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2510_05254_b200 as ndgx
for arith in (ndgx.ARITH_EXACT, ndgx.ARITH_FAST):
    mesh = ndgx.Mesh(2, (12, 10), 8)
    model = ndgx.EquationModel.isothermal_euler(2, 1.0)
    u0 = ndgx.init_euler_subsonic(mesh, model)
    with ndgx.Solver(ndgx.SolverConfig(mesh, model, ndgx.RK4, 0.4, 1.0), device=0, arith=arith) as s:
        s.upload(u0); print("upload ok", flush=True)
        r = s.rhs(); print("rhs ok", np.abs(r).max(), flush=True)
        st = s.advance(ndgx.StepPlan(3, False)); print("advance ok", st, flush=True)
