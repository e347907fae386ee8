"""Build a tuning variant of libndgx.so that differs only in the 2D order-8
contracted-arithmetic kernels (the flagship): _variants/<name>/libndgx.so.

    python scripts/variant.py NAME [-DMACRO=VALUE ...]

Run with NDGX_LIB=_variants/<name>/libndgx.so.  The other objects come from
paper_2510_05254_b200/_build (python -m paper_2510_05254_b200.build first).
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05254_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "_variants", name)
os.makedirs(out, exist_ok=True)
dims = os.environ.get("VARIANT_INST", "2,8,0").split(";")
objs = [o for o in glob.glob(os.path.join(b.BUILD, "*.o"))]
for inst in dims:
    d, n, e = inst.split(",")
    tag = f"ndgx_inst_d{d}_o{n}_e{e}"
    obj = os.path.join(out, tag + ".o")
    cmd = [b.NVCC] + b.ARCH + b.FLAGS + [f"-DNDGX_DIM={d}", f"-DNDGX_ORDER={n}", f"-DNDGX_EXACT={e}"] + flags + \
        ["-c", os.path.join(b.CSRC, "ndgx_inst.cu"), "-o", obj]
    subprocess.run(cmd, check=True)
    objs = [o for o in objs if os.path.basename(o) != tag + ".o"] + [obj]
# slim library: the other instances are stubs returning "not compiled" (small
# enough to ship to the GPU box next to the others)
keep = {f"ndgx_inst_d{i.split(',')[0]}_o{i.split(',')[1]}_e{i.split(',')[2]}" for i in dims}
stub = os.path.join(out, "stubs.cu")
with open(stub, "w") as f:
    f.write('#include "ndgx_kernels.h"\nnamespace ndgx {\n')
    for d in (1, 2, 3):
        for n in range(2, 9):
            for e in (0, 1):
                if f"ndgx_inst_d{d}_o{n}_e{e}" not in keep:
                    f.write(f"StageKernel NDGX_ENTRY_NAME({d}, {n}, {e})(int) {{ return StageKernel{{}}; }}\n")
    f.write("}\n")
subprocess.run([b.NVCC] + b.ARCH + b.FLAGS + ["-c", stub, "-o", stub + ".o"], check=True)
objs = [o for o in objs if not os.path.basename(o).startswith("ndgx_inst_") or os.path.basename(o)[:-2] in keep]
subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-o", os.path.join(out, "libndgx.so")] + objs + [stub + ".o", "-lpthread", "-ldl"],
               check=True)
for o in glob.glob(os.path.join(out, "*.o")) + [stub]:
    os.remove(o)
print(os.path.join(out, "libndgx.so"))
