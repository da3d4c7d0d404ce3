"""The drop-in, end to end: the maintainer's binding
`process_frame_b200` (oracle/ref/pipeline_b200.cpp), compiled against the
reference's own headers and linked with the unmodified reference objects and
libstitch_b200.so into oracle/_ref/integration_demo.  The demo runs the
reference's stitch::initialize, copies the PipelineState, and drives one copy
through stitch::process_frame (the reference, CPU) and the other through the
binding (the B200 path): panoramas, masks, colour matrices (bitwise), rank
flags, thresholds and frame indices must be identical on every frame.
The binary is built here (where /root/reference exists) and travels to the
GPU box prebuilt."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "integration_demo")


def _need_demo():
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/integration_demo not built (needs /root/reference)")


def test_binding_links_the_in_tree_library():
    _need_demo()
    out = subprocess.run(["ldd", DEMO], capture_output=True, text=True).stdout
    line = [ln for ln in out.splitlines() if "libstitch_b200.so" in ln]
    assert line and "not found" not in line[0]
    assert os.path.realpath(line[0].split("=>")[1].split("(")[0].strip()) == os.path.realpath(
        os.path.join(ROOT, "paper_2308_09209_b200", "libstitch_b200.so"))


@pytest.mark.gpu
@pytest.mark.parametrize("views,w,h,frames,refine,masked", [(2, 640, 480, 12, 1, 0),
                                                            (3, 320, 240, 6, 1, 0),
                                                            (2, 320, 240, 5, 0, 0),
                                                            (2, 640, 480, 6, 1, 1),
                                                            (3, 320, 240, 4, 0, 1),
                                                            (2, 320, 240, 5, 1, 2),
                                                            (3, 320, 240, 5, 0, 2)])
def test_binding_reproduces_reference_process_frame(views, w, h, frames, refine, masked):
    """masked: every frame (the first ones included) carries a Frame::mask;
    masked = 2 also masks frame 2 of the last view completely, where the
    reference throws EmptyProjection and the binding must throw it too."""
    _need_demo()
    r = subprocess.run([DEMO, str(views), str(w), str(h), str(frames), str(refine), "0",
                        str(masked)],
                       capture_output=True, text=True, timeout=900)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert lines, r.stdout[-2000:] + r.stderr[-2000:]
    res = json.loads(lines[-1])
    print(lines[-1])
    assert r.returncode == 0 and res["identical"], res
    assert res["errors"] == (1 if masked == 2 else 0), res
