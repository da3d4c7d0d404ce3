"""bench.py --gpus N launches N ranks itself (RANK / LOCAL_RANK / WORLD_SIZE /
MASTER_*), the driver's contract for the scaling run, and refuses a --gpus
that disagrees with an outer launcher's WORLD_SIZE.  CPU: the reference arm
(rank 0 alone prints; the other ranks exit 0).  GPU: the B200 arm with two
ranks on the one box (ranks share the device round-robin and report
"oversubscribed"; a functional check of the multi-rank path, not a scaling
number)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "MASTER_ADDR",
              "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=e,
                          capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def test_gpus_two_spawns_ranks_reference_arm():
    p = _run(["--gpus", "2", "--impl", "reference", "--config", "c1", "--steps", "1",
              "--warmup", "0", "--no-calibration"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    res = json.loads(lines[0])
    assert res["impl"] == "reference" and res["steps"] == 1


def test_gpus_mismatch_with_world_size_fails_loudly():
    p = _run(["--gpus", "2", "--impl", "reference", "--config", "c1", "--steps", "1"],
             env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode != 0 and "WORLD_SIZE" in (p.stderr + p.stdout)


@pytest.mark.gpu
def test_gpus_two_b200_arm_reports_aggregate():
    p = _run(["--gpus", "2", "--steps", "5", "--warmup", "3", "--e2e-steps", "5",
              "--no-cpu-baseline"], timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    res = json.loads(lines[0])
    assert res["n_gpus"] == 2 and res["config"]["streams_total"] == 2
    assert res["value"] > 0 and res["e2e"]["value"] > 0


@pytest.mark.gpu
def test_c5_sixty_four_streams_sharded_over_two_ranks():
    p = _run(["--gpus", "2", "--config", "c5", "--steps", "3", "--warmup", "3",
              "--e2e-steps", "3", "--frame-sets", "2", "--no-cpu-baseline"], timeout=1200)
    assert p.returncode == 0, p.stderr[-3000:]
    res = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][0])
    assert res["scaling"] == "strong" and res["config"]["streams_total"] == 64
    assert res["config"]["streams_this_rank"] == 32


@pytest.mark.gpu
def test_both_arms_report_the_same_workload_geometry():
    """The reference arm (the compiled reference on c1) and the B200 arm name
    the same workload: same canvas, pair bounds and refined pairs, computed
    independently by each arm's own initialize."""
    ref = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"])
    gpu = _run(["--config", "c1", "--steps", "3", "--warmup", "3", "--e2e-steps", "3",
                "--no-cpu-baseline"], timeout=900)
    assert ref.returncode == 0 and gpu.returncode == 0, ref.stderr[-2000:] + gpu.stderr[-2000:]
    rc = json.loads([ln for ln in ref.stdout.splitlines() if ln.startswith("{")][-1])["config"]
    gc = json.loads([ln for ln in gpu.stdout.splitlines() if ln.startswith("{")][-1])["config"]
    for key in ("workload", "config_key", "cameras", "camera_size", "canvas", "pairs",
                "refined_pairs"):
        assert rc[key] == gc[key], (key, rc[key], gc[key])
