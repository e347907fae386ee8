import sys, time, json
sys.path.insert(0, ".")
import numpy as np
import paper_2510_05254_b200 as ndgx
out = {}
for arith in ([int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else (ndgx.ARITH_EXACT, ndgx.ARITH_FAST)):
    cases = [(2,(768,768),8,1,ndgx.RK4), (3,(128,128,128),4,1,ndgx.RK6), (2,(388,388),8,0,ndgx.RK4)]
    if len(sys.argv) > 2 and sys.argv[2] == "3d":  # the 3D order-4 shape under every integrator
        cases = [(3,(128,128,128),4,1,rk) for rk in (ndgx.RK3, ndgx.RK4, ndgx.RK6)]
    for (dim, cells, order, eq, rk) in cases:
        mesh = ndgx.Mesh(dim, cells, order)
        model = ndgx.EquationModel.isothermal_euler(dim,1.0) if eq else ndgx.EquationModel.advection(dim,(1,0,0))
        u0 = ndgx.init_euler_subsonic(mesh, model) if eq else ndgx.init_multisine(mesh, model, n_modes=40, seed=42)
        with ndgx.Solver(ndgx.SolverConfig(mesh, model, rk), arith=arith) as s:
            s.upload(u0)
            s.advance(ndgx.StepPlan(3, True))
            st = s.advance(ndgx.StepPlan(20, False))
            prof = s.profile_step()
            v = s.dof * s.stages * st.steps / st.wall_seconds
            key = f"{dim}D eq{eq} o{order} rk{rk} arith{arith}"
            out[key] = dict(dofstage_per_s=v, ms_per_step=st.wall_seconds/st.steps*1e3, stage_ms=prof[0], ctl_ms=prof[1])
            print(key, json.dumps(out[key]), flush=True)
