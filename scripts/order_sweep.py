"""Throughput across (dim, order, equation) at ~1e8 DOF, fast arithmetic (tuning / evidence).

    python scripts/order_sweep.py [tag] > out.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_05254_b200 as ndgx  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "main"
arith = ndgx.ARITH_EXACT if (len(sys.argv) > 2 and sys.argv[2] == "exact") else ndgx.ARITH_FAST
cases = [(2, o, 1) for o in range(2, 9)] + [(2, o, 0) for o in range(2, 9)] + \
        [(1, o, 0) for o in (2, 4, 6, 8)] + [(3, o, 1) for o in (2, 3, 4, 5)] + [(3, o, 0) for o in (2, 3)]
if len(sys.argv) > 3:  # dim:order:eq,...
    cases = [tuple(int(x) for x in c.split(":")) for c in sys.argv[3].split(",")]
for dim, order, eq in cases:
    target = 1.0e8
    nv = (dim + 1) if eq else 1
    per_cell = order ** dim * nv
    c = max(4, int(round((target / per_cell) ** (1.0 / dim))))
    cells = (c,) * dim
    mesh = ndgx.Mesh(dim, cells, order)
    model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if eq else ndgx.EquationModel.advection(dim, (1, 0.5, 0.25))
    cfg = ndgx.SolverConfig(mesh, model, ndgx.RK4, 0.4, 1.0)
    with ndgx.Solver(cfg, arith=arith) as s:
        s.init_device(ndgx.IC_EULER_SUBSONIC if eq else ndgx.IC_MULTISINE,
                      None if eq else ndgx.multisine_amplitudes(4, 1))
        s.advance(ndgx.StepPlan(3, True))
        best = None
        for _ in range(2):
            st = s.advance(ndgx.StepPlan(10, False))
            ms = st.wall_seconds / st.steps * 1e3
            best = ms if best is None else min(best, ms)
        v = s.dof * s.stages / best * 1e3
        print(json.dumps({"tag": tag, "dim": dim, "order": order, "eq": "euler" if eq else "adv",
                          "cells": list(cells), "dof": s.dof, "ms_per_step": round(best, 4),
                          "dofstage_per_s": v, "hbm_frac_26B": v * 26 / 1e9 / 6545.9}), flush=True)
