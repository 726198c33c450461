"""Aggregate an ncu CSV of one forward (scripts/ncu_forward.py): per kernel
class time share, DRAM bytes and achieved GB/s, tensor-pipe utilisation
(duration-weighted), and the forward total (serialised by ncu)."""
import collections
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
k = collections.OrderedDict()
for r in rows[hi + 1:]:
    kid = r[idi]
    d = k.setdefault(kid, {"name": re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")})
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(unit, 1)
    d[r[mi]] = v * scale
cls = collections.OrderedDict()
tot_t = tot_b = tc_w = 0.0
for d in k.values():
    n = d["name"]
    c = "gemm" if "gemm" in n else "attention" if "attn" in n else n.split("_kernel")[0]
    t = d.get("gpu__time_duration.sum", 0.0)
    b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tc = d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
    e = cls.setdefault(c, {"n": 0, "time_us": 0.0, "dram_mb": 0.0, "tensor_pct_time_weighted": 0.0})
    e["n"] += 1
    e["time_us"] += t * 1e6
    e["dram_mb"] += b / 1e6
    e["tensor_pct_time_weighted"] += tc * t
    tot_t += t
    tot_b += b
    tc_w += tc * t
for e in cls.values():
    e["gbs"] = e["dram_mb"] / e["time_us"] * 1e3 if e["time_us"] else 0.0
    e["tensor_pct_time_weighted"] = e["tensor_pct_time_weighted"] / (e["time_us"] * 1e-6) if e["time_us"] else 0.0
    e["share"] = e["time_us"] / (tot_t * 1e6)
out = {"kernels": len(k), "time_us": tot_t * 1e6, "dram_mb": tot_b / 1e6, "dram_gbs": tot_b / tot_t / 1e9,
       "tensor_pct_time_weighted": tc_w / tot_t, "classes": cls}
print(json.dumps(out, indent=1))
