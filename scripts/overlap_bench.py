"""Cost of the halo exchange on one B200: ms/step of the single-block solver
against the same mesh run as exchanging blocks.

    python scripts/overlap_bench.py [fast|exact]

Cases: C3 through the NCCL rank path with every axis forced through the
transport (world size 1); C3 as one forced-exchange block of the
partitioned handle; C3 as 2 / 4 partitioned blocks; a C5 P=8-sized block
pair (2048 x 512 cells, decompose -> two 1024 x 512 blocks, x-split).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_05254_b200 as ndgx  # noqa: E402

arith = ndgx.ARITH_EXACT if (len(sys.argv) > 1 and sys.argv[1] == "exact") else ndgx.ARITH_FAST
steps = 20 if not (len(sys.argv) > 2 and sys.argv[2] == "3d") else 4


def timed(s, u0):
    s.upload(u0)
    s.advance(ndgx.StepPlan(3, True))
    best = None
    for _ in range(3):
        st = s.advance(ndgx.StepPlan(steps, False))
        ms = st.wall_seconds / st.steps * 1e3
        best = ms if best is None else min(best, ms)
    stage = s.profile_step()[0]
    return best, [round(x, 4) for x in stage]


def case(name, cells, variants, order=8, rk=ndgx.RK4):
    dim = len(cells)
    mesh = ndgx.Mesh(dim, cells, order)
    model = ndgx.EquationModel.isothermal_euler(dim, 1.0)
    cfg = ndgx.SolverConfig(mesh, model, rk, 0.4, 1.0)
    u0 = ndgx.init_euler_subsonic(mesh, model)
    with ndgx.Solver(cfg, arith=arith) as s:
        base, bst = timed(s, u0)
    print(json.dumps({"case": name, "variant": "single block", "ms_per_step": round(base, 4), "stage_ms": bst}),
          flush=True)
    for label, make in variants:
        with make(cfg) as s:
            ms, st = timed(s, u0)
        print(json.dumps({"case": name, "variant": label, "ms_per_step": round(ms, 4), "stage_ms": st,
                          "vs_single": round(ms / base, 4)}), flush=True)


case("C3 768^2", (768, 768), [
    ("rank path, NCCL self-exchange on both axes",
     lambda c: ndgx.Solver.for_rank(c, 1, 0, ndgx.nccl_unique_id(), arith=arith, force_exchange=True)),
    ("partitioned P=1, both axes through the halo planes",
     lambda c: ndgx.Solver.partitioned(c, 1, arith=arith, force_exchange=True)),
    ("partitioned P=2 (1,2,1)", lambda c: ndgx.Solver.partitioned(c, 2, arith=arith)),
    ("partitioned P=4 (2,2,1)", lambda c: ndgx.Solver.partitioned(c, 4, arith=arith)),
])
case("C5/8-sized blocks 2048x512", (2048, 512), [
    ("partitioned P=2 (2,1,1): two 1024x512 blocks", lambda c: ndgx.Solver.partitioned(c, 2, arith=arith)),
])
if len(sys.argv) > 2 and sys.argv[2] == "3d":
    # the C4 weak-scaling shape at N = 2: two 128^3 z-slabs (decompose -> (1, 1, 2))
    case("C4 x2 128x128x256 (3D Euler o4 RK6)", (128, 128, 256), [
        ("partitioned P=2 (1,1,2): two 128^3 z-slabs", lambda c: ndgx.Solver.partitioned(c, 2, arith=arith)),
    ], order=4, rk=ndgx.RK6)
