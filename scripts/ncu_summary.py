"""Summarise an ncu --set full report (.ncu-rep) into the numbers the
profiles/ notes cite: duration, DRAM bytes, IPC, occupancy, top stall
reasons, instruction mix.  Usage: python scripts/ncu_summary.py rep [...]"""
import csv
import io
import subprocess
import sys
from collections import Counter

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
       "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
       "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed.avg.per_cycle_active", "lts__t_bytes.sum"]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(rep):
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        lines.append(f"kernel: {name}")
        for k in RAW:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"  {k:62s} {r[i]} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
                    "_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):
                                                  -len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        lines.append("  stall reasons (warps per issue): " +
                     ", ".join(f"{n} {v:.2f}" for v, n in stalls[:8]))
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    if len(src) > 2:
        h = src[1]
        ie, sc = h.index("Instructions Executed"), h.index("Source")
        mix = Counter()
        tot = 0
        for r in src[2:]:
            if len(r) <= max(ie, sc) or not r[ie].isdigit():
                continue
            t = r[sc].split()
            op = (t[1] if t and t[0].startswith("@") else t[0]).split(".")[0] if t else "?"
            mix[op] += int(r[ie])
            tot += int(r[ie])
        lines.append(f"  warp instructions executed: {tot}")
        lines.append("  mix: " + ", ".join(f"{o} {n / tot * 100:.1f}%" for o, n in mix.most_common(12)))
    return "\n".join(lines)


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(f"== {rep}")
        print(summarise(rep))
