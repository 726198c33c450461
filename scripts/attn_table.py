"""Table of attn_tc_kernel times from attn_bench.py ncu logs: per config the
median of the warm launches, TF/s and fraction of the bf16 burst peak."""
import csv
import json
import re
import sys
from pathlib import Path

peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["bf16_tflops"]
for csv_path in sys.argv[1:]:
    log = Path(csv_path).with_suffix(".log").read_text()
    cfgs = re.findall(r"H=(\d+) C=(\d+): attention ([\d.]+) GFLOP", log)
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ts = [float(r[h.index("Metric Value")].replace(",", "")) for r in rows[hi + 1:]
          if r[h.index("Metric Name")] == "gpu__time_duration.sum"]
    # launches per config: prefill launches (ceil(H/8192)) then 3 chunk launches
    i = 0
    for H, C, gf in cfgs:
        H = int(H)
        i += (H + 8191) // 8192
        chunk = sorted(ts[i:i + 3][1:])
        i += 3
        us = chunk[len(chunk) // 2] / 1e3 if chunk else float("nan")
        tf = float(gf) * 1e9 / (us * 1e-6) / 1e12
        print(f"{Path(csv_path).stem:28s} H={H:6d} C={C}: {us:8.1f} us  {tf:7.1f} TF/s  {tf / peak:.2f} of burst")
