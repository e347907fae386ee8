"""Per-source-line memory traffic from an ncu source page CSV: L1 tag requests
(global), shared wavefronts (+ excessive), L2 theoretical sectors (+ excessive).

    python scripts/ncu_mem_lines.py src.csv [top] [elements]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
elems = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
hdr = None
cur_file = None
out = []
tot = {}
keys = ["L1 Tag Requests Global", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive",
        "L2 Theoretical Sectors Global", "L2 Theoretical Sectors Global Excessive", "Instructions Executed"]
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0]:
        continue
    d = dict(zip(hdr, r))
    vals = {}
    for k in keys:
        try:
            vals[k] = float(d.get(k, "0") or 0)
        except ValueError:
            vals[k] = 0.0
        tot[k] = tot.get(k, 0.0) + vals[k]
    w = vals["L1 Tag Requests Global"] + vals["L1 Wavefronts Shared"]
    if w > 0:
        out.append((w, cur_file, r[0], r[1].strip()[:80], vals))
print("per element totals:", {k: round(v / elems, 1) for k, v in tot.items()})
for w, f, ln, src, v in sorted(out, reverse=True)[:top]:
    print(f"{w / elems:8.1f} {f}:{ln:>5} tagG={v['L1 Tag Requests Global'] / elems:6.1f} "
          f"wfS={v['L1 Wavefronts Shared'] / elems:6.1f} (exc {v['L1 Wavefronts Shared Excessive'] / elems:5.1f}) "
          f"L2sec={v['L2 Theoretical Sectors Global'] / elems:6.1f} (exc {v['L2 Theoretical Sectors Global Excessive'] / elems:5.1f}) | {src}")
