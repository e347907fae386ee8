"""Registers / stack / spills per stage-kernel instance from `nvcc -Xptxas -v` output.

    python scripts/ptxas_table.py DIM ORDER EXACT [extra nvcc flags...]
"""
import re
import subprocess
import sys

dim, order, exact = sys.argv[1:4]
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
       "-I", "include", "-I", "paper_2510_05254_b200/csrc", f"-DNDGX_DIM={dim}", f"-DNDGX_ORDER={order}",
       f"-DNDGX_EXACT={exact}", "-Xptxas", "-v", "-c", "paper_2510_05254_b200/csrc/ndgx_inst.cu", "-o", "/tmp/_pt.o"]
cmd += sys.argv[4:]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows.setdefault(cur, {})["stack/spill"] = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows.setdefault(cur, {})["regs"] = m.group(1)
for k, v in rows.items():
    m = re.search(r"stage_kernelILi(\d)ELi(\d)ELi(\d)ELb(\d)ELi(\d)E", k)
    if not m:
        continue
    print(f"dim{m.group(1)} N{m.group(2)} kind{m.group(3)} exact{m.group(4)} sig{m.group(5)}: "
          f"regs {v.get('regs')} stack/spill-st/spill-ld {v.get('stack/spill')}")
