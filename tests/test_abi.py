"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
function include/stitch_b200.h declares, and the ctypes structs match the
header layout.  No compute calls (no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2308_09209_b200 as pb
from paper_2308_09209_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stitch_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stitch_b200_\w+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _abi.load()
    names = declared_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    # and the ctypes table covers the header
    assert sorted(n for n, _, _ in _abi.SYMBOLS) == names


SYNTH_HEADER = os.path.join(ROOT, "include", "stitch_synth.h")


def test_synth_library_is_separate():
    """the input generator (stitch_synth.h) lives in libstitch_synth.so, which
    exports exactly its C API; the product library exports none of it."""
    src = re.sub(r"/\*.*?\*/", "", open(SYNTH_HEADER).read(), flags=re.S)
    names = sorted(set(re.findall(r"\b(stitch_b200_synth_\w+)\s*\(", src)))
    assert names and sorted(n for n, _, _ in _abi.SYNTH_SYMBOLS) == names
    synth = subprocess.run(["nm", "-D", "--defined-only", _abi.SYNTH_LIB_PATH],
                           capture_output=True, text=True, check=True).stdout
    assert sorted(set(re.findall(r" T (\w+)", synth))) == names
    prod = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True,
                          text=True, check=True).stdout
    assert "stitch_b200_synth_" not in prod
    _abi.load_synth()


def test_exported_dynamic_symbols():
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (stitch_b200_\w+)", out))
    assert set(declared_functions()) <= exported


def test_struct_layouts_match_header():
    # compile a tiny C program against the header and compare sizeof/offsetof
    prog = r"""
#include <stdio.h>
#include <stddef.h>
#include "stitch_synth.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(stitch_b200_camera), sizeof(stitch_b200_config),
   sizeof(stitch_b200_pair), sizeof(stitch_b200_init), sizeof(stitch_b200_report),
   sizeof(stitch_b200_synth_spec), offsetof(stitch_b200_init, pairs));
 return 0; }
"""
    tmp = "/tmp/stitch_b200_layout"
    with open(tmp + ".c", "w") as f:
        f.write(prog)
    subprocess.run(["/usr/bin/gcc", "-I", os.path.join(ROOT, "include"), tmp + ".c", "-o", tmp],
                   check=True)
    got = [int(x) for x in subprocess.run([tmp], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [C.sizeof(_abi.Camera), C.sizeof(_abi.Config), C.sizeof(_abi.Pair),
            C.sizeof(_abi.Init), C.sizeof(_abi.Report), C.sizeof(_abi.SynthSpec),
            _abi.Init.pairs.offset]
    assert got == want


def test_config_defaults_match_reference():
    lib = _abi.load()
    c = _abi.Config()
    lib.stitch_b200_config_defaults(C.byref(c))
    # BalanceConfig (color_balance.hpp:19-25), FlowOptions (flow.hpp:29-34),
    # window 3 / fuse "own" (pipeline.hpp:39-42)
    assert (c.lambda_, c.gamma_dark, c.gamma_bright) == (0.05, 1.5, 1.5)
    assert (c.target_black, c.target_white) == (0, 255)
    assert (c.flow_levels, c.flow_iterations, c.smoothness) == (4, 50, 15.0)
    # refinement on (pipeline.hpp:24)
    assert (c.window_capacity, c.fuse_weighting, c.refine_enabled) == (3, 0, 1)
    assert pb.RefineOptions().enabled is True


def test_mirror_defaults_match_reference():
    """the Python mirror's StitchConfig equals the compiled reference's
    StitchConfig defaults (pipeline.hpp:17-45) field by field."""
    import oracle.reference as R

    if not R.available():
        pytest.skip("reference neither present nor prebuilt")
    o = R.default_opts()
    cfg = pb.StitchConfig()
    assert (cfg.balance.lambda_, cfg.balance.gamma_dark, cfg.balance.gamma_bright,
            cfg.balance.target_black, cfg.balance.target_white) == (
        o.lambda_, o.gamma_dark, o.gamma_bright, o.target_black, o.target_white)
    assert (cfg.flow.levels, cfg.flow.iterations, cfg.flow.smoothness) == (
        o.levels, o.iterations, o.smoothness)
    assert (cfg.window_capacity, cfg.fuse_weighting == "cross", cfg.threads) == (
        o.window_capacity, bool(o.fuse_weighting), o.threads)
    r = cfg.refine
    assert (r.enabled, r.margin, r.ransac_iters, r.inlier_px, r.detect_threshold, r.match_ratio,
            r.rerefine_every) == (bool(o.refine_enabled), o.refine_margin, o.ransac_iters,
                                  o.inlier_px, o.detect_threshold, o.match_ratio,
                                  o.rerefine_every)


def test_last_error_is_a_string():
    lib = _abi.load()
    assert isinstance(lib.stitch_b200_last_error(), bytes)
    assert b"sm_100a" in lib.stitch_b200_version()


def test_missing_library_fails_loudly(tmp_path):
    _abi._lib_saved = _abi._lib
    try:
        _abi._lib = None
        with pytest.raises(ImportError):
            _abi.load(str(tmp_path / "nope.so"))
    finally:
        _abi._lib = _abi._lib_saved


@pytest.mark.parametrize("workers", [0, 1, 3, 14])
def test_host_copy_pool_back_to_back_batches(workers):
    """The pool that stages pageable frames: thousands of back-to-back
    batches (the submit / wait pattern), every byte checked -- a late worker
    must never touch a finished batch (host only, no GPU needed)."""
    lib = _abi.load()
    assert lib.stitch_b200_debug_copy_pool(workers, 3000, 3 << 20) == 0, lib.stitch_b200_last_error()
