"""File ingress / egress throughput at BASELINE config C2 (4 x 1080p):
stitch_b200_run_files over numbered PPM sequences (16 pre-rendered frame
sets, later frames hard-linked to them so the page cache holds the inputs),
panoramas written as PPM.  Reports frames/s with and without the writes and
the summed per-file read / write times.
Usage: python scripts/bench_files.py [frames] [out.json]"""
import json
import os
import shutil
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2308_09209_b200 as pb  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 120
out_json = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/files_c2.json"
base = "/dev/shm" if os.path.isdir("/dev/shm") else None
root = tempfile.mkdtemp(prefix="stitch_files_", dir=base)
try:
    wl = bench.WORKLOADS["c2"]
    sc = bench.build_scene(wl, 1)
    dirs = []
    for v in range(wl["views"]):
        d = os.path.join(root, f"view{v}")
        os.makedirs(d)
        for t in range(frames):
            name = os.path.join(d, pb.sequence_name("cam", t, ".ppm"))
            if t < 16:
                pb.write_ppm(name, sc.render_view(v, t))
            else:
                os.link(os.path.join(d, pb.sequence_name("cam", t % 16, ".ppm")), name)
        dirs.append(d)
    state = pb.initialize(sc.config(), [sc.render_view(v, 0) for v in range(wl["views"])])
    pb.run_files(state, dirs, None, max_frames=8)  # warm-up
    ingress = pb.run_files(state, dirs, None)
    out_dir = os.path.join(root, "out")
    full = pb.run_files(state, dirs, out_dir)
    canvas = state.canvas
    state.close()
    res = {
        "workload": wl["desc"], "frames": frames, "storage": base or tempfile.gettempdir(),
        "read_only": {"fps": round(ingress.fps(), 1), "seconds": round(ingress.seconds, 3),
                      "read_seconds_summed": round(ingress.read_seconds, 3)},
        "read_write": {"fps": round(full.fps(), 1), "seconds": round(full.seconds, 3),
                       "read_seconds_summed": round(full.read_seconds, 3),
                       "write_seconds_summed": round(full.write_seconds, 3)},
        "bytes_per_frame": {"ppm_in": 4 * (1920 * 1080 * 3 + 15),
                            "ppm_out": canvas[0] * canvas[1] * 3},
    }
    print(json.dumps(res))
    os.makedirs(os.path.dirname(os.path.abspath(out_json)), exist_ok=True)
    with open(out_json, "w") as f:
        json.dump(res, f, indent=1)
finally:
    shutil.rmtree(root, ignore_errors=True)
