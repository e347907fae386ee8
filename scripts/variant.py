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
subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-o", os.path.join(out, "libndgx.so")] + objs + ["-lpthread", "-ldl"],
               check=True)
for o in glob.glob(os.path.join(out, "*.o")):
    os.remove(o)
print(os.path.join(out, "libndgx.so"))
