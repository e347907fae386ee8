"""Bitwise comparison of final states across _variants libraries (tuning check).

    python scripts/cmp_variants.py OUTDIR   (run once per NDGX_LIB, then --compare)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_05254_b200 as ndgx  # noqa: E402

out = sys.argv[1]
if len(sys.argv) > 2 and sys.argv[2] == "--compare":
    import glob
    files = sorted(glob.glob(os.path.join(out, "*.npy")))
    groups = {}
    for f in files:
        tag, case = os.path.basename(f)[:-4].split("__")
        groups.setdefault(case, []).append((tag, np.load(f)))
    for case, arrs in groups.items():
        base_tag, base = arrs[0]
        for tag, a in arrs[1:]:
            d = np.max(np.abs(a - base)) if a.shape == base.shape else -1
            print(f"{case}: {tag} vs {base_tag}: equal={np.array_equal(a, base)} maxdiff={d:.3e}")
    sys.exit(0)
tag = os.path.basename(os.path.dirname(os.environ.get("NDGX_LIB", "main/x")))
os.makedirs(out, exist_ok=True)
mesh = ndgx.Mesh(3, (4, 4, 16), 4)
model = ndgx.EquationModel.isothermal_euler(3, 1.0)
cfg = ndgx.SolverConfig(mesh, model, ndgx.RK6, 0.4, 1.0)
u0 = ndgx.init_euler_subsonic(mesh, model)
for steps in (1, 7):
    with ndgx.Solver(cfg, arith=ndgx.ARITH_FAST) as s:
        s.upload(u0)
        s.advance(ndgx.StepPlan(steps, True))
        np.save(os.path.join(out, f"{tag}__single{steps}.npy"), s.download())
    with ndgx.Solver.partitioned(cfg, 4, arith=ndgx.ARITH_FAST) as s:
        s.upload(u0)
        s.advance(ndgx.StepPlan(steps, True))
        np.save(os.path.join(out, f"{tag}__part{steps}.npy"), s.download())
print("saved", tag)
