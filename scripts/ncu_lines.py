"""Aggregate an ncu report's per-source-line metrics (instructions executed,
warp stall samples) from `ncu -i REP --page source --csv --print-source
cuda,sass`; prints the top lines.  Usage: ncu_lines.py REP [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
path = fn = None
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        iw, ie = 4, 7  # Warp Stall Sampling (All Samples), Instructions Executed
        try:
            w, e = int(r[iw] or 0), int(r[ie] or 0)
        except ValueError:
            continue
        key = (path, int(r[0]))
        a = agg.setdefault(key, [0, 0, r[1][:90]])
        a[0] += e
        a[1] += w
te = sum(a[0] for a in agg.values()) or 1
tw = sum(a[1] for a in agg.values()) or 1
print(f"instructions {te}, stall samples {tw}")
for (p, ln), (e, w, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{p}:{ln:<5d} instr {100 * e / te:5.1f}%  stalls {100 * w / tw:5.1f}%  {src}")
