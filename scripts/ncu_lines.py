"""Per-source-line stall summary from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
cur_file, cur_line, cur_src = None, None, None
agg = defaultdict(lambda: defaultdict(float))
srcs = {}
total = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if not r[0]:
        continue  # SASS rows; the source-line row carries the aggregate
    cur_line, cur_src = r[0], r[1]
    srcs[(cur_file, cur_line)] = cur_src.strip()[:90]
    key = (cur_file, cur_line)
    d = {k: (v if v not in ("-", "") else "0") for k, v in zip(hdr[2:], r[2:])}
    try:
        s = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
    except ValueError:
        continue
    total += s
    agg[key]["samples"] += s
    agg[key]["inst"] += float(d.get("Instructions Executed", 0) or 0)
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                agg[key][k] += float(v)
            except ValueError:
                pass
items = sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]
print(f"total samples {total:.0f}")
for (f, ln), d in items:
    stalls = sorted(((k[6:], v) for k, v in d.items() if k.startswith("stall_")), key=lambda x: -x[1])[:3]
    st = " ".join(f"{k}={v/max(d['samples'],1):.0%}" for k, v in stalls if v > 0)
    print(f"{d['samples']/total:6.1%} {f}:{ln:>4} inst={d['inst']:.0f} [{st}] {srcs.get((f, ln), '')}")
