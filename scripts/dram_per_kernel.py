"""Per-kernel achieved DRAM bandwidth of one frame from an ncu launch list
with gpu__time_duration.sum, dram__bytes_read.sum and dram__bytes_write.sum
(cold caches, serialised launches): measured bytes / measured time against
the measured HBM peak (MEASURED_PEAKS.json).  Usage:
  python scripts/dram_per_kernel.py launches.csv [out.txt]"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = collections.defaultdict(dict)
order = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    key = int(r["ID"])
    if key not in rows:
        order.append(key)
    rows[key]["name"] = r["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1].split("<")[0]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "byte": 1, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    rows[key][r["Metric Name"]] = v * scale
idx = [k for k in order if rows[k]["name"].startswith("k_expand")]
frame = [k for k in order if idx[-2] <= k < idx[-1]]
try:
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    peak = 6650.0
agg = collections.OrderedDict()
for k in frame:
    r = rows[k]
    a = agg.setdefault(r["name"], [0, 0.0, 0.0])
    a[0] += 1
    a[1] += r.get("gpu__time_duration.sum", 0.0)
    a[2] += r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
out = [f"{'kernel':18s} {'launches':>8s} {'us/frame':>9s} {'DRAM MB':>9s} {'GB/s':>8s} {'% of peak':>9s}"]
for name, (n, t, b) in agg.items():
    gbs = b / t / 1e9 if t > 0 else 0.0
    out.append(f"{name:18s} {n:8d} {t * 1e6:9.1f} {b / 1e6:9.1f} {gbs:8.1f} {100 * gbs / peak:8.1f}%")
tt = sum(a[1] for a in agg.values())
tb = sum(a[2] for a in agg.values())
out.append(f"{'frame':18s} {len(frame):8d} {tt * 1e6:9.1f} {tb / 1e6:9.1f} {tb / tt / 1e9:8.1f} "
           f"{100 * tb / tt / 1e9 / peak:8.1f}%   (peak {peak:.1f} GB/s)")
text = "\n".join(out)
print(text)
if len(sys.argv) > 2:
    with open(sys.argv[2], "w") as f:
        f.write(text + "\n")
