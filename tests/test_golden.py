"""Golden fixtures (tests/golden/oracle_small.json, made by
tests/golden/make_golden.py): SHA-256 digests of the oracle's outputs on
small fixed scenes.  CPU: the oracle still produces them.  GPU: the B200 path
produces the same digests (panorama RGB + mask, colour matrices, rank flags,
thresholds, both flow fields of every pair) without consulting the oracle."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2308_09209_b200 as pb
from paper_2308_09209_b200 import _abi
from tests.golden.make_golden import CASES, case_digest, sha
from tests.helpers import frames_at, product_config, scene

GOLDEN = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                     "oracle_small.json")))


@pytest.mark.parametrize("name,skw,ckw,frames", CASES, ids=[c[0] for c in CASES])
def test_oracle_reproduces_golden(name, skw, ckw, frames):
    assert case_digest(scene(**skw), ckw, frames) == GOLDEN["cases"][name]


@pytest.mark.gpu
@pytest.mark.parametrize("name,skw,ckw,frames", CASES, ids=[c[0] for c in CASES])
def test_b200_matches_golden(name, skw, ckw, frames):
    want = GOLDEN["cases"][name]
    sc = scene(**skw)
    state = pb.initialize(product_config(sc, **ckw), frames_at(sc, 0))
    lib = _abi.load()
    try:
        assert list(state.canvas) == want["canvas"] and len(state.pairs) == want["pairs"]
        for t in range(frames):
            res = pb.process_frame(state, frames_at(sc, t))
            fw = want["frames"][t]
            assert sha(res.panorama.data) == fw["pano_rgb"], (name, t)
            assert sha(res.panorama.mask) == fw["pano_mask"], (name, t)
            rep = res.report
            assert [sha(np.asarray(m, np.float64).reshape(9)) for m in rep.color_matrices] == fw["m"]
            assert [int(x) for x in rep.rank_deficient] == fw["rank_deficient"]
            assert list(rep.threshold_m1) == fw["m1"] and list(rep.threshold_m2) == fw["m2"]
            flows = []
            for k, p in enumerate(state.pairs):
                shape = (p.bounds[3] - p.bounds[1], p.bounds[2] - p.bounds[0])
                for d in range(2):
                    u = np.zeros(shape, np.float32)
                    v = np.zeros(shape, np.float32)
                    pb.pipeline.check(lib.stitch_b200_debug_flow(state.handle, k, d,
                                                                 u.ctypes.data_as(C.c_void_p),
                                                                 v.ctypes.data_as(C.c_void_p)))
                    flows.append(sha(np.stack([u, v])))
            assert flows == fw["flows"], (name, t)
    finally:
        state.close()
