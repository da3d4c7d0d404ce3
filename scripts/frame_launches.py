"""Print the kernel launches of one frame from an ncu launch-list CSV
(scripts/launch_list.sh): the launches between the last two k_expand
launches, with the per-kind totals."""
import collections
import csv
import sys

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r["Metric Name"] == "gpu__time_duration.sum":
        rows.append((r["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1], r["Grid Size"],
                     float(r["Metric Value"]) / 1e3))
idx = [i for i, r in enumerate(rows) if r[0].startswith("k_expand")]
frame = rows[idx[-2]:idx[-1]]
tot = collections.OrderedDict()
for name, grid, us in frame:
    if "-v" in sys.argv:
        print(f"{name:40s} {grid:14s} {us:8.1f}")
    key = name.split("<")[0]
    tot[key] = tot.get(key, 0.0) + us
for k, v in tot.items():
    print(f"{k:24s} {v:8.1f} us")
print(f"{'frame':24s} {sum(v for _, _, v in frame):8.1f} us, {len(frame)} launches")
