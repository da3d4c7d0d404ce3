"""Measurement (GPU box): the contract-tolerant Jacobi sweep
(STITCH_B200_HS_FAST=1: FMA contraction and the approximate reciprocal instead
of the reference's unfused arithmetic and IEEE division) against the oracle at
BASELINE.json's full sizes, C1-C4, checked against north_star's contract --
flows within 1e-3 px, colour matrices within 1e-4 relative, panoramas within
+-1 LSB, masks, thresholds and rank flags identical.  Each config runs in a
subprocess (the switch is read once per process) and prints its max diffs
as one RESULT JSON line; profiles/r02_fast_sweep_contract.json records the
outcome (the variant breaks the contract, so the bit-exact sweep stays).

    python -m pytest scripts/fast_sweep_contract.py -q -s
    CONTRACT_ENV=STITCH_B200_WARP_F32=1 python -m pytest scripts/fast_sweep_contract.py -q -s

CONTRACT_ENV (comma-separated NAME=VALUE, default STITCH_B200_HS_FAST=1) picks the
contract-tolerant variant under test.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import json, sys
from tests.fullsize import run_config
key = sys.argv[1]
geom, frames, info = run_config(key)
worst = {"config": key, "geometry_equal": geom, "frames": len(frames),
         "flow_max_abs_px": max(d["flow_max_abs_px"] for d in frames),
         "color_matrix_max_rel": max(d["color_matrix_max_rel"] for d in frames),
         "panorama_max_abs_lsb": max(d["panorama_max_abs_lsb"] for d in frames),
         "mask_equal": all(d["mask_equal"] for d in frames),
         "thresholds_equal": all(d["thresholds_equal"] for d in frames),
         "rank_flags_equal": all(d["rank_flags_equal"] for d in frames)}
print("RESULT " + json.dumps(worst))
"""


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["c1", "c2", "c3", "c4"])
def test_fast_sweep_within_contract(key):
    spec = os.environ.get("CONTRACT_ENV", "STITCH_B200_HS_FAST=1")
    env = dict(os.environ, **dict(kv.split("=", 1) for kv in spec.split(",") if kv))
    r = subprocess.run([sys.executable, "-c", CODE, key], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    d = json.loads(line[len("RESULT "):])
    print(line)
    assert d["geometry_equal"]
    assert d["flow_max_abs_px"] <= 1e-3, d
    assert d["color_matrix_max_rel"] <= 1e-4, d
    assert d["panorama_max_abs_lsb"] <= 1, d
    assert d["mask_equal"] and d["thresholds_equal"] and d["rank_flags_equal"], d
