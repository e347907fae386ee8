import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2510_05254_b200 as ndgx
T0 = time.time()
def log(*a): print(f"[{time.time()-T0:7.1f}]", *a, flush=True)
cases = [(2, (12, 10), 8, True, ndgx.RK4), (3, (4, 6, 5), 4, True, ndgx.RK6), (2, (9, 7), 3, False, ndgx.RK3), (1, (64,), 4, False, ndgx.RK4)]
for dim, cells, order, euler, rk in cases:
    mesh = ndgx.Mesh(dim, cells, order)
    model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if euler else ndgx.EquationModel.advection(dim, (1, 0, 0))
    cfg = ndgx.SolverConfig(mesh, model, rk, 0.4, 1.0)
    u0 = ndgx.init_euler_subsonic(mesh, model) if euler else ndgx.init_multisine(mesh, model, n_modes=5, seed=3)
    with ndgx.Solver(cfg) as s:
        s.upload(u0); rw = s.rhs(); stw = s.advance(ndgx.StepPlan(7, True)); want = s.download()
    log("serial done", dim, cells, order)
    nid = ndgx.nccl_unique_id(); log("uid")
    s = ndgx.Solver.for_rank(cfg, 1, 0, nid, force_exchange=True); log("create", list(s.plan.split))
    s.upload(u0); r = s.rhs(); log("rhs", np.array_equal(r, rw), np.abs(r-rw).max())
    st = s.advance(ndgx.StepPlan(7, True)); got = s.download(); log("adv", np.array_equal(got, want), st.steps, stw.steps)
    s.close(); log("closed")
