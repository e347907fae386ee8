"""Per-stage DRAM traffic of the stage kernels from ncu summaries -> profiles/ncu_stage_traffic.json
(bench.py's roofline.traffic).

    python scripts/traffic_table.py c3=profiles/r02/final_ncu_c3.json c4=... c2=...
"""
import json
import os
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {}
for arg in sys.argv[1:]:
    cfg, path = arg.split("=", 1)
    rows = json.load(open(path))
    per = []
    for k in rows:
        b = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = k[key].split()
            b += float(v) * UNIT[u]
        per.append(b)
    out[cfg] = {"fast": {"dram_bytes_per_launch": sum(per) / len(per), "per_stage": per,
                         "source": f"ncu --set full, the stage kernels of one step ({os.path.relpath(path, ROOT)})"}}
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_stage_traffic.json"), "w"), indent=1)
print(json.dumps({c: v["fast"]["dram_bytes_per_launch"] for c, v in out.items()}))
