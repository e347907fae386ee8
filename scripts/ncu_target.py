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
dim, cells, order, eq, rk, desc = CONFIGS[name]
mesh = ndgx.Mesh(dim, cells, order)
model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if eq else ndgx.EquationModel.advection(dim, (1, 0, 0))
u0 = ndgx.init_euler_subsonic(mesh, model) if eq else ndgx.init_multisine(mesh, model, n_modes=40, seed=42)
with ndgx.Solver(ndgx.SolverConfig(mesh, model, rk), arith=arith) as s:
    s.upload(u0)
    st = s.advance(ndgx.StepPlan(steps, False))
    print(desc, "arith", sys.argv[2] if len(sys.argv) > 2 else "exact", "steps", st.steps,
          "ms/step", st.wall_seconds / st.steps * 1e3)
