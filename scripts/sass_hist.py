"""SASS instruction histograms of the hot stage kernels (static counts from cuobjdump).

    python scripts/sass_hist.py OUT.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_2510_05254_b200", "_build")
# (object, dim, order, kind, exact, sigs, note)
KERNELS = [("ndgx_inst_d2_o8_e0.o", 2, 8, 1, 0, (0, 1, 3), "C3 flagship: 2D Euler o8 RK4 (DMMA body)"),
           ("ndgx_inst_d2_o8_e0.o", 2, 8, 0, 0, (0, 1, 3), "C2: 2D advection o8 RK4 (DMMA body)"),
           ("ndgx_inst_d3_o4_e0.o", 3, 4, 1, 0, (0, 1, 4, 5, 6, 7, 8), "C4: 3D Euler o4 RK6 (DMMA body)"),
           ("ndgx_inst_d2_o8_e1.o", 2, 8, 1, 1, (0, 1, 3), "C3 exact mode (generic body)"),
           ("ndgx_inst_d2_o4_e0.o", 2, 4, 1, 0, (0, 1, 3), "2D Euler o4 (generic body, 8 lanes per element)"),
           ("ndgx_inst_d2_o7_e0.o", 2, 7, 1, 0, (0, 1, 3), "2D Euler o7 (flagship body zero-padded to 8 x 8)")]
KEYS = ["DMMA", "DFMA", "DMUL", "DADD", "MUFU", "LDG", "STG", "LDS", "STS", "LDL", "STL", "UBLKCP", "LDGSTS",
        "SYNCS", "SHFL", "BAR", "WARPSYNC", "BRA", "BSSY", "IMAD", "ISETP", "LOP3"]


def main(out):
    lines = ["# SASS instruction histograms (static, per kernel; `cuobjdump -sass`, sm_100a)", "",
             "Columns count instructions in the kernel's SASS listing (not dynamic executions).",
             "LDL/STL = local-memory (spill/stack) traffic; UBLKCP = TMA bulk copies; DMMA = FP64 tensor-core MMA.",
             ""]
    for obj, d, n, kind, ex, sigs, note in KERNELS:
        path = os.path.join(BUILD, obj)
        lines += [f"## {note}", "", "| sig | total | " + " | ".join(KEYS) + " |",
                  "|---|---|" + "---|" * len(KEYS)]
        for sig in sigs:
            sym = f"_ZN4ndgx12stage_kernelILi{d}ELi{n}ELi{kind}ELb{ex}ELi{sig}ELb0EEEvNS_9StageArgsE"
            sass = subprocess.run(["cuobjdump", "-sass", "-fun", sym, path], capture_output=True, text=True).stdout
            ops = re.findall(r"^\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", sass, re.M)
            base = collections.Counter(o.split(".")[0] for o in ops)
            lines.append(f"| {sig} | {sum(base.values())} | " + " | ".join(str(base.get(k, 0)) for k in KEYS) + " |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02/sass_hist.md")
