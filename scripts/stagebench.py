"""Per-stage times (in-graph stamps) and graph-timed ms/step for C3 / C2 (fast).

    NDGX_LIB=... python scripts/stagebench.py [tag] [configs, default c3,c2]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_05254_b200 as ndgx  # noqa: E402
from bench import CONFIGS  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("NDGX_LIB", "default")
names = (sys.argv[2] if len(sys.argv) > 2 else "c3,c2").split(",")
for name in names:
    dim, cells, order, eq, rk, desc = CONFIGS[name]
    mesh = ndgx.Mesh(dim, cells, order)
    model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if eq else ndgx.EquationModel.advection(dim, (1, 0, 0))
    u0 = ndgx.init_euler_subsonic(mesh, model) if eq else ndgx.init_multisine(mesh, model, n_modes=40, seed=42)
    with ndgx.Solver(ndgx.SolverConfig(mesh, model, rk), arith=ndgx.ARITH_FAST) as s:
        s.upload(u0)
        s.advance(ndgx.StepPlan(3, True))
        best = None
        for _ in range(3):
            st = s.advance(ndgx.StepPlan(20 if name != "c4" else 4, False))
            ms = st.wall_seconds / st.steps * 1e3
            best = ms if best is None else min(best, ms)
        reps = int(os.environ.get("STAGEBENCH_REPS", "3"))
        stage = None
        for _ in range(reps):  # per-stage minimum over repeated in-graph profiles (box noise ~5%)
            prof = s.profile_step()[0]
            stage = prof if stage is None else [min(a, b) for a, b in zip(stage, prof)]
        print(json.dumps({"tag": tag, "cfg": name, "ms_per_step": round(best, 4),
                          "dofstage_per_s": s.dof * s.stages / best * 1e3,
                          "stage_ms": [round(x, 4) for x in stage]}), flush=True)
