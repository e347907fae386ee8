import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2510_05254_b200 as ndgx
print("start", flush=True)
mesh = ndgx.Mesh(2, (12, 10), 8); model = ndgx.EquationModel.isothermal_euler(2, 1.0)
cfg = ndgx.SolverConfig(mesh, model)
u0 = ndgx.init_euler_subsonic(mesh, model)
nid = ndgx.nccl_unique_id(); print("uid ok", flush=True)
s = ndgx.Solver.for_rank(cfg, 1, 0, nid, force_exchange=True); print("create ok", list(s.plan.split), flush=True)
s.upload(u0); print("upload ok", flush=True)
r = s.rhs(); print("rhs ok", flush=True)
st = s.advance(ndgx.StepPlan(3, False)); print("advance ok", st, flush=True)
s.close(); print("done", flush=True)
