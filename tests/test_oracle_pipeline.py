"""Pipeline-level properties of the CPU oracle, restating the reference's
specified (unshipped) pipeline tests: SPEC.md:517-519 (steady state,
flicker harness), :526 / :531 (thread-count determinism), :532 (causality),
:160-162 (window length 1 == 2D-M).  CPU only, small sizes."""
import numpy as np

import oracle as O
from tests.helpers import frames_at, oracle_config, scene


def run(sc, frames, **kw):
    st = O.OracleState(oracle_config(sc, **kw))
    out = [st.process([f.data for f in frames_at(sc, t)]) for t in range(frames)]
    st.close()
    return out


def test_static_scene_steady_state_bit_identical_from_frame_3():
    sc = scene(views=2, width=120, height=90, obj=False)
    out = run(sc, 5)
    for t in range(3, 5):
        np.testing.assert_array_equal(out[t][0], out[2][0])
        np.testing.assert_array_equal(out[t][1], out[2][1])


def test_thread_count_determinism():  # SPEC.md:526, pipeline.hpp:87-89
    sc = scene(views=3, width=120, height=90)
    a = run(sc, 2, threads=1)
    b = run(sc, 2, threads=4)
    for (da, ma, _), (db, mb, _) in zip(a, b):
        np.testing.assert_array_equal(da, db)
        np.testing.assert_array_equal(ma, mb)


def test_causality_prefix():
    sc = scene(views=2, width=120, height=90)
    a = run(sc, 3)
    b = run(sc, 2)
    for t in range(2):
        np.testing.assert_array_equal(a[t][0], b[t][0])


def test_window_one_is_2dm():  # SPEC.md:160, color_transfer.hpp window capacity 1
    sc = scene(views=2, width=120, height=90, casts=[(1, 1, 1), (0.8, 1.0, 1.1)])
    w1 = run(sc, 3, window=1)
    # window 1 at frame t == a fresh pipeline (empty window) fed frame t alone
    for t in range(1, 3):
        st = O.OracleState(oracle_config(sc, window=1))
        st.process([f.data for f in frames_at(sc, t)])
        _, _, rep = st.process([f.data for f in frames_at(sc, t)])
        np.testing.assert_array_equal(np.array(rep.m[0][:]), np.array(w1[t][2].m[0][:]))


def test_flicker_damped_by_temporal_window():  # SPEC.md:519 (Table 2 sigma)
    flick = [dict(frame=3, view=1, gains=(1.3, 1.3, 1.3))]
    import paper_2308_09209_b200 as pb

    sc = scene(views=2, width=120, height=90, obj=False, casts=[(1, 1, 1), (0.9, 1, 1.05)],
               flicker=[pb.FlickerEvent(**f) for f in flick])

    def jump(window):
        # how much the per-frame correction M moves between consecutive frames
        out = run(sc, 6, window=window)
        ms = [np.array(o[2].m[0][:]) for o in out]
        return max(np.abs(ms[t] - ms[t - 1]).max() for t in range(1, 6))

    assert jump(3) < jump(1)


def test_chain_topology_reduces_to_star_for_three_views():
    sc = scene(views=3, width=120, height=90)
    a = run(sc, 2, topology=0)
    b = run(sc, 2, topology=1)
    for (da, _, _), (db, _, _) in zip(a, b):
        np.testing.assert_array_equal(da, db)


def test_four_view_chain_runs_and_pairs_are_adjacent():
    sc = scene(views=4, width=120, height=90)
    st = O.OracleState(oracle_config(sc))
    pairs = [st.pair(k)[:2] for k in range(st.n_pairs())]
    ref = sc.reference_view()
    assert ref == 1
    assert pairs == [(0, 1), (2, 1), (3, 2)]
    data, mask, rep = st.process([f.data for f in frames_at(sc, 0)])
    assert mask.sum() > 0 and rep.balanced == 1


def test_ring_rig_oracle_geometry():
    """360-degree ring extension: cylindrical canvas spans 2*pi*f, pairs form
    a ring chain outward from the reference, the opposite view straddles the
    canvas seam, and a frame stitches with every pixel column covered."""
    import math

    import paper_2308_09209_b200 as pb

    sc = pb.SynthScene(pb.SynthSpec(views=6, width=192, height=108, rig="ring"))
    st = O.OracleState(oracle_config(sc))
    c = sc.config_c()
    w, h, ox, oy = st.canvas
    assert w == math.ceil(2 * math.pi * c.cyl_focal)
    pairs = [st.pair(k)[:2] for k in range(st.n_pairs())]
    assert pairs == [(1, 0), (5, 0), (2, 1), (4, 5), (3, 2)]
    x0, _, x1, _ = st.view_bbox(3)
    assert x0 == 0 and x1 == w  # wraps around the seam
    data, mask, rep = st.process([f.data for f in frames_at(sc, 0)])
    assert mask.any(axis=0).all() and rep.balanced == 1
