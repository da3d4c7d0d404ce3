"""The reference's error behaviour on masked inputs that warp to nothing,
pinned to THE REFERENCE ITSELF (tests/golden/reference_errors.json, made by
tests/golden/make_reference_errors.py from the compiled reference).

warp_frame throws EmptyProjection when a view has no valid warped pixel
(geometry.cpp:79).  process_frame warps first (pipeline.cpp:270-277), so the
frame fails with the temporal state untouched and the following frames match
a run that never saw it; initialize fails the same way on a fully masked
first frame (rebuild_pair_geometry, pipeline.cpp:181-188).

* CPU: the oracle reproduces every error and every digest around them;
* GPU: the B200 path does -- process_frame (stitch_b200_process_masked)
  raises EmptyProjection before the frame is enqueued, the pipelined
  submit path likewise, and initialize on a fully masked first frame.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2308_09209_b200 as pb
from tests.golden.masks import case_masks
from tests.test_ref_pin import first_diff, frame_digest, oracle_state, product_scene, product_state

GOLDEN = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                     "reference_errors.json")))
CASES = list(GOLDEN["cases"].items())
IDS = [c[0] for c in CASES]
EMPTY_PROJECTION = 10  # stitch::ErrorCode::EmptyProjection (types.hpp:9-27)


def masks_at(case, t):
    s = case["scene"]
    return [case_masks(s["masks"], v, t, s["width"], s["height"]) for v in range(s["views"])]


def test_golden_errors_are_empty_projection():
    for name, case in CASES:
        codes = [case["init_error"]] if "init_error" in case else \
            [f["error"] for f in case["frames"] if "error" in f]
        assert codes and set(codes) == {EMPTY_PROJECTION}, name


@pytest.mark.parametrize("name,case", CASES, ids=IDS)
def test_oracle_reproduces_reference_errors(name, case):
    sc = product_scene(case["scene"])
    nv = case["scene"]["views"]
    first = [sc.render_view(v, 0).data for v in range(nv)]
    try:
        if "init_error" in case:
            with pytest.raises(O.OracleError) as ei:
                oracle_state(sc, case["opts"], first, masks_at(case, 0))
            assert ei.value.code == case["init_error"]
            return
        ost = oracle_state(sc, case["opts"], first, masks_at(case, 0))
        try:
            assert list(ost.canvas) == case["canvas"]
            for t, want in enumerate(case["frames"]):
                frames = [sc.render_view(v, t).data for v in range(nv)]
                if "error" in want:
                    with pytest.raises(O.OracleError) as ei:
                        ost.process(frames, masks_at(case, t))
                    assert ei.value.code == want["error"], (name, t)
                    continue
                data, mask, rep = ost.process(frames, masks_at(case, t))
                got = frame_digest(data, mask, [rep.m[k][:] for k in range(rep.n_pairs)],
                                   [rep.rank_deficient[k] for k in range(rep.n_pairs)],
                                   rep.threshold_m1, rep.threshold_m2)
                assert first_diff(got, want, t) is None, (name, first_diff(got, want, t))
        finally:
            ost.close()
    finally:
        sc.close()


def _frames(sc, case, t):
    nv = case["scene"]["views"]
    ms = masks_at(case, t)
    return [pb.Frame(sc.render_view(v, t).data, ms[v]) for v in range(nv)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,case", CASES, ids=IDS)
def test_b200_reproduces_reference_errors(name, case):
    sc = product_scene(case["scene"])
    try:
        if "init_error" in case:
            with pytest.raises(pb.StitchError) as ei:
                product_state(sc, case["opts"], _frames(sc, case, 0))
            assert ei.value.code == pb.ErrorCode(case["init_error"]), name
            return
        state = product_state(sc, case["opts"], _frames(sc, case, 0))
        try:
            assert [state.canvas_width, state.canvas_height] == case["canvas"][:2]
            for t, want in enumerate(case["frames"]):
                if "error" in want:
                    with pytest.raises(pb.StitchError) as ei:
                        pb.process_frame(state, _frames(sc, case, t))
                    assert ei.value.code == pb.ErrorCode(want["error"]), (name, t)
                    continue
                res = pb.process_frame(state, _frames(sc, case, t))
                r = res.report
                got = frame_digest(res.panorama.data, res.panorama.mask, r.color_matrices,
                                   r.rank_deficient, r.threshold_m1, r.threshold_m2)
                assert first_diff(got, want, t) is None, (name, first_diff(got, want, t))
        finally:
            state.close()
    finally:
        sc.close()


@pytest.mark.gpu
def test_b200_pipelined_submit_skips_the_failed_frame():
    """stitch_b200_submit_masked with frames in flight: the fully masked frame
    is refused at submit (no ticket), the frames before and after it keep
    their tickets and the reference's digests."""
    import ctypes as C

    from paper_2308_09209_b200 import _abi

    name = "frame_empty"
    case = GOLDEN["cases"][name]
    lib = _abi.load()
    sc = product_scene(case["scene"])
    state = product_state(sc, case["opts"], _frames(sc, case, 0))
    try:
        w, h = state.canvas_width, state.canvas_height
        nv = case["scene"]["views"]
        keep, tickets = [], {}
        for t, want in enumerate(case["frames"]):
            fr = _frames(sc, case, t)
            arrs = [np.ascontiguousarray(f.data) for f in fr]
            ms = [None if f.mask is None else np.ascontiguousarray(f.mask, np.uint8) for f in fr]
            rgb = np.zeros((h, w, 3), np.uint8)
            mask = np.zeros((h, w), np.uint8)
            keep.append((arrs, ms, rgb, mask))
            ptrs = (C.c_void_p * nv)(*[a.ctypes.data for a in arrs])
            mptrs = (C.c_void_p * nv)(*[None if m is None else m.ctypes.data for m in ms])
            tk = C.c_longlong(-1)
            rc = lib.stitch_b200_submit_masked(state.handle, ptrs, mptrs, rgb.ctypes.data,
                                               mask.ctypes.data, C.byref(tk))
            if "error" in want:
                assert rc == want["error"] + 1, (t, rc)
                continue
            assert rc == 0, (t, rc)
            tickets[t] = tk.value
        for t, tk in tickets.items():
            rep = _abi.Report()
            pb.pipeline.check(lib.stitch_b200_wait(state.handle, tk, C.byref(rep)))
            r = pb.pipeline._report_from_c(rep)
            _, _, rgb, mask = keep[t]
            got = frame_digest(rgb, mask, r.color_matrices, r.rank_deficient, r.threshold_m1,
                               r.threshold_m2)
            assert first_diff(got, case["frames"][t], t) is None, (t, first_diff(got, case["frames"][t], t))
    finally:
        state.close()
        sc.close()
