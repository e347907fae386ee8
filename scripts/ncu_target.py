"""Small driver for ncu captures: builds one solver and runs a few fixed steps.

    python scripts/ncu_target.py [c3|c2|c4|c5] [exact|fast] [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_05254_b200 as ndgx  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
arith = ndgx.ARITH_FAST if (len(sys.argv) > 2 and sys.argv[2] == "fast") else ndgx.ARITH_EXACT
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if name in CONFIGS:
    dim, cells, order, eq, rk, desc = CONFIGS[name]
else:  # dim:order:eq at ~1e8 DOF, RK4 (order sweeps)
    dim, order, eq = (int(x) for x in name.split(":"))
    c = max(4, int(round((1e8 / (order ** dim * ((dim + 1) if eq else 1))) ** (1.0 / dim))))
    cells, rk, desc = (c,) * dim, 1, f"{dim}D order {order} eq {eq}, {c}^{dim} cells"

mesh = ndgx.Mesh(dim, cells, order)
model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if eq else ndgx.EquationModel.advection(dim, (1, 0, 0))
with ndgx.Solver(ndgx.SolverConfig(mesh, model, rk), arith=arith) as s:
    s.init_device(ndgx.IC_EULER_SUBSONIC if eq else ndgx.IC_MULTISINE, None if eq else ndgx.multisine_amplitudes(40, 42))
    st = s.advance(ndgx.StepPlan(steps, False))
    print(desc, "arith", sys.argv[2] if len(sys.argv) > 2 else "exact", "steps", st.steps,
          "ms/step", st.wall_seconds / st.steps * 1e3)
