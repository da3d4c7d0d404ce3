"""profiles/traffic.json from an ncu launch list (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum): DRAM bytes per launch of each
kernel kind bench.py profiles, averaged over one C2 frame's launches.  A kind
whose op is two kernels (statistics + solve, canvas + LUT) counts both per op.
Usage: python scripts/traffic_json.py profiles/r02_launches.csv profiles/traffic.json"""
import collections
import csv
import json
import sys

KINDS = {  # bench.py kind: (kernels of one op, the kernel counted once per op)
    "expand_rgba": (("k_expand",), "k_expand"),
    "crop_warp": (("k_crop_warp",), "k_crop_warp"),
    "pair_color": (("k_pair_color", "k_pair_solve"), "k_pair_color"),
    "flow_prepare": (("k_flow_prepare_pyr",), "k_flow_prepare_pyr"),
    "hs_sweeps": (("k_hs_sweep",), "k_hs_sweep"),
    "hs_linearize": (("k_hs_linearize",), "k_hs_linearize"),
    "canvas_balance": (("k_canvas", "k_balance"), "k_canvas"),
    "tone": (("k_tone",), "k_tone"),
}


def main():
    src, out = sys.argv[1], sys.argv[2]
    lines = [ln for ln in open(src) if ln.startswith('"')]
    rows = collections.defaultdict(dict)
    order = []
    for r in csv.DictReader(lines):
        k = int(r["ID"])
        if k not in rows:
            order.append(k)
        rows[k]["name"] = (r["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0]
                           .split("::")[-1])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1)
        rows[k][r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * scale
    idx = [k for k in order if rows[k]["name"] == "k_expand"]
    frame = [k for k in order if idx[-2] <= k < idx[-1]]
    note = (f"ncu launch list of one C2 frame (dram__bytes_read.sum + dram__bytes_write.sum, "
            f"cold caches, serialised), {src}; averaged over the frame's launches of this kernel "
            f"(a two-kernel op counts both)")
    res = {}
    for kind, (names, per_op) in KINDS.items():
        b = sum(rows[k].get("dram__bytes_read.sum", 0) + rows[k].get("dram__bytes_write.sum", 0)
                for k in frame if rows[k]["name"] in names)
        n = sum(1 for k in frame if rows[k]["name"] == per_op)
        if n:
            res[kind] = {"dram_bytes_per_launch": int(round(b / n)), "launches_per_frame": n,
                         "source": note}
    json.dump(res, open(out, "w"), indent=1)
    print({k: v["dram_bytes_per_launch"] for k, v in res.items()})


if __name__ == "__main__":
    main()
