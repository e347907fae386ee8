"""Generate tests/golden/ fixtures by running the REFERENCE itself.

Requires oracle/_ref/libndg_ref.so, built from /root/reference/proj/src by
``make -C oracle ref`` (this container only; /root/reference is absent on the
GPU box, so the fixtures are committed).  Run:

    python tests/golden/make_golden.py

Writes golden.json (digests, norms, step statistics, error messages) and
golden_states.npz (small full states in the reference AoS layout).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import (ADVECTION, EULER, RK3, RK4, RK6, CheckerError, Oracle,  # noqa: E402
                        Problem, fnv1a64)

# (name, problem, ic, fixed_steps, t_end-mode, store-state)
CASES = [
    # SURVEY.md appendix KATs (reference -O3, StepPlan{100,false})
    ("adv1d_o4_rk4_1024", Problem(1, (1024,), 4, ADVECTION, RK4), {"amps": [1.0]}, 100, False),
    ("adv2d_o8_rk4_48", Problem(2, (48, 48), 8, ADVECTION, RK4), {"n_modes": 40, "seed": 42}, 100, False),
    ("euler2d_o8_rk4_48", Problem(2, (48, 48), 8, EULER, RK4), {}, 100, False),
    ("euler3d_o4_rk6_12", Problem(3, (12, 12, 12), 4, EULER, RK6), {}, 100, False),
    # small full-state fixtures over the (dim, order, model, scheme) grid
    ("adv1d_o2_rk3_16", Problem(1, (16,), 2, ADVECTION, RK3), {"n_modes": 3, "seed": 7}, 20, True),
    ("adv1d_o8_rk6_10", Problem(1, (10,), 8, ADVECTION, RK6), {"n_modes": 2, "seed": 5}, 20, True),
    ("adv2d_o3_rk4_6x5", Problem(2, (6, 5), 3, ADVECTION, RK4, velocity=(1.0, -0.5, 0.0)),
     {"n_modes": 4, "seed": 9}, 10, True),
    ("adv2d_o5_rk3_4x7", Problem(2, (4, 7), 5, ADVECTION, RK3, velocity=(0.3, 0.8, 0.0)),
     {"n_modes": 2, "seed": 1}, 10, True),
    ("adv3d_o2_rk3_4", Problem(3, (4, 4, 4), 2, ADVECTION, RK3), {"n_modes": 2, "seed": 5}, 6, True),
    ("adv3d_o4_rk4_3x4x5", Problem(3, (3, 4, 5), 4, ADVECTION, RK4, velocity=(0.5, 1.0, -0.25)),
     {"n_modes": 3, "seed": 11}, 8, True),
    ("euler2d_o3_rk4_8", Problem(2, (8, 8), 3, EULER, RK4), {}, 8, True),
    ("euler2d_o4_rk6_5x6", Problem(2, (5, 6), 4, EULER, RK6, sound_speed=1.3), {}, 10, True),
    ("euler2d_o8_rk3_4x3", Problem(2, (4, 3), 8, EULER, RK3), {}, 10, True),
    ("euler2d_o7_rk4_3", Problem(2, (3, 3), 7, EULER, RK4, length=(2.0, 1.5, 1.0)), {}, 10, True),
    ("euler3d_o3_rk4_4", Problem(3, (4, 4, 4), 3, EULER, RK4), {}, 10, True),
    ("euler3d_o4_rk6_3x4x2", Problem(3, (3, 4, 2), 4, EULER, RK6), {}, 6, True),
    ("euler3d_o2_rk3_5x3x4", Problem(3, (5, 3, 4), 2, EULER, RK3), {}, 10, True),
]

T_END_CASES = [
    # (name, problem, ic) run with StepPlan{-1, false}: t_end landing semantics
    ("tend_adv1d_o4_10", Problem(1, (10,), 4, ADVECTION, RK4, t_end=1.0), {"n_modes": 2, "seed": 5}),
    ("tend_adv2d_o3_6", Problem(2, (6, 6), 3, ADVECTION, RK4, t_end=0.03), {"n_modes": 3, "seed": 7}),
    ("tend_short_adv1d", Problem(1, (8,), 3, ADVECTION, RK4, t_end=0.004), {"amps": [1.0]}),
    ("tend_euler2d_o4_6", Problem(2, (6, 6), 4, EULER, RK3, t_end=0.05), {}),
    ("tend_zero_wavespeed", Problem(1, (8,), 3, ADVECTION, RK4, velocity=(0.0, 0.0, 0.0), t_end=0.7),
     {"amps": [0.5]}),
]


def problem_dict(p: Problem) -> dict:
    return {"dim": p.dim, "cells": list(p.cells3), "order": p.order, "kind": p.kind, "rk": p.rk,
            "velocity": list(p.velocity), "sound_speed": p.sound_speed, "cfl": p.cfl,
            "t_end": p.t_end, "length": list(p.length)}


def make_initial(ref: Oracle, p: Problem, ic: dict) -> np.ndarray:
    if p.kind == EULER:
        return ref.init_euler(p)
    if "amps" in ic:
        return ref.init_multisine(p, amps=ic["amps"])
    return ref.init_multisine(p, n_modes=ic["n_modes"], seed=ic["seed"])


def main() -> None:
    ref = Oracle("reference")
    out = {"generator": "tests/golden/make_golden.py", "checker": "oracle/_ref/libndg_ref.so",
           "cases": {}, "t_end": {}, "errors": {}, "decompose": []}
    states = {}
    for name, p, ic, steps, store in CASES:
        u0 = make_initial(ref, p, ic)
        r0 = ref.rhs(p, u0)
        uf, st = ref.advance(p, u0, steps, False)
        zero = np.zeros_like(uf)
        out["cases"][name] = {
            "problem": problem_dict(p), "ic": ic, "fixed_steps": steps,
            "digest_init": fnv1a64(u0), "digest_rhs0": fnv1a64(r0), "digest_final": fnv1a64(uf),
            "l2_final": [ref.l2_error(p, uf, zero, v) for v in range(p.n_var)],
            "steps": st.steps, "dt_min": st.dt_min, "dt_max": st.dt_max,
            "rhs0_first": float(r0[0]),
        }
        if store:
            states[name + "/init"] = u0
            states[name + "/rhs0"] = r0
            states[name + "/final"] = uf
        print(name, out["cases"][name]["digest_final"], st.steps)
    for name, p, ic in T_END_CASES:
        u0 = make_initial(ref, p, ic)
        uf, st = ref.advance(p, u0, -1, False)
        out["t_end"][name] = {"problem": problem_dict(p), "ic": ic, "steps": st.steps,
                              "dt_min": st.dt_min, "dt_max": st.dt_max,
                              "digest_final": fnv1a64(uf)}
        states[name + "/init"] = u0
        states[name + "/final"] = uf
        print(name, st.steps, st.dt_max)

    # error semantics (test_solver.cpp:239-255, 380-394; solver.cpp:411-413)
    p = Problem(2, (4, 4), 3, EULER, RK4)
    u = ref.init_euler(p)
    idx = ((2 * 4 + 1) * 3 * 3 + (1 * 3 + 1)) * 3 + 0  # cell (2,1), node (1,1), rho
    u[idx] = -0.5
    states["err_rho/init"] = u
    for what, fn in (("rhs", lambda: ref.rhs(p, u)), ("advance", lambda: ref.advance(p, u, 4))):
        try:
            fn()
            raise SystemExit("expected PhysicsError")
        except CheckerError as e:
            out["errors"]["negative_density_" + what] = {"code": e.code, "step": e.step,
                                                         "message": e.message}
    p = Problem(1, (8,), 3, ADVECTION, RK4)
    u = ref.init_multisine(p, amps=[1.0])
    u[3] = float("nan")
    states["err_nan/init"] = u
    try:
        ref.advance(p, u, -1)
        raise SystemExit("expected InstabilityError")
    except CheckerError as e:
        out["errors"]["nan_state"] = {"code": e.code, "step": e.step, "message": e.message}
    p = Problem(1, (8,), 3, ADVECTION, RK4, velocity=(0.0, 0.0, 0.0))
    try:
        ref.advance(p, ref.init_multisine(p, amps=[0.5]), 3)
        raise SystemExit("expected ConfigError")
    except CheckerError as e:
        out["errors"]["zero_wavespeed_fixed"] = {"code": e.code, "step": e.step, "message": e.message}

    # decompose KATs (test_partition.cpp:33-125 plus the bench grids)
    for dim, cells, workers in [(2, (100, 100), 4), (2, (100, 10), 10), (2, (8, 8), 2),
                                (2, (7, 5), 1), (3, (128, 128, 256), 2), (3, (128, 128, 1024), 8),
                                (2, (2048, 2048), 8), (2, (2048, 2048), 2), (2, (2048, 2048), 4),
                                (3, (256, 256, 256), 8), (3, (4, 5, 6), 6), (1, (13,), 3)]:
        pp = Problem(dim, cells, 2, ADVECTION)
        grid, lo, hi, nbr = ref.decompose(pp, workers)
        out["decompose"].append({"dim": dim, "cells": list(pp.cells3), "workers": workers,
                                 "grid": list(grid), "lo": lo.tolist(), "hi": hi.tolist(),
                                 "nbr": nbr.tolist()})

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden_states.npz"), **states)


if __name__ == "__main__":
    main()
