"""Max-abs-diff report of the B200 path against the CPU oracle at the
BASELINE.json configurations (bench inputs), per stage and per frame.
Usage: python scripts/parity_report.py [out.json] [config ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests.fullsize import run_config  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_report.json"
keys = sys.argv[2:] or ["c1", "c2", "c3", "c4"]
report = []
for key in keys:
    geom, frames, info = run_config(key)
    worst = {k: (max(f[k] for f in frames) if not isinstance(frames[0][k], bool)
                 else all(f[k] for f in frames)) for k in frames[0]}
    report.append({**info, "init_geometry_equal": geom, "worst": worst, "per_frame": frames})
    print(json.dumps({"config": key, "init_geometry_equal": geom, "worst": worst}))
os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
with open(out, "w") as f:
    json.dump(report, f, indent=1)
