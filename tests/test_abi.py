"""The C-ABI library loads and exports every symbol include/aps.h declares;
host-only entry points (no device) behave as documented.  CPU only."""
import ctypes
import os
import re

import numpy as np
import pytest

import synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def aps():
    from paper_1911_08907_b200 import build
    build.build()
    import paper_1911_08907_b200 as pkg
    pkg.load()
    return pkg


def _declared():
    src = open(os.path.join(ROOT, "include", "aps.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(aps_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(aps):
    declared = _declared()
    assert len(declared) >= 25
    L = aps.load()
    for name in declared:
        assert hasattr(L, name), name
    from paper_1911_08907_b200.aps import EXPORTS
    assert sorted(EXPORTS) == declared


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_1911_08907_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "liboracle" not in text, f
                assert "from oracle" not in text, f


def test_layout_matches_oracle(aps, orc):
    for numels in (synthetic.C1_NUMELS, synthetic.RESNET50_NUMELS, [1], [127, 129, 1, 5000]):
        for p in (1, 2, 3, 4, 8):
            for e, m in [(5, 2), (3, 0), (5, 6), (5, 10), (8, 23)]:
                T, nb = aps.layout(p, e, m, numels)
                assert T == orc.total_tiles(p, numels)
                assert nb == orc.packed_bytes(p, e, m, numels)


def test_layout_mixed_matches_oracle(aps, orc):
    """Per-layer formats (aps_layout_mixed) against the oracle's mixed layout;
    uniform formats reduce to aps_layout."""
    rng = np.random.default_rng(5)
    fmts_all = [(5, 2), (3, 0), (4, 3), (5, 6), (5, 10), (8, 23), (2, 1)]
    for numels in (synthetic.C1_NUMELS, synthetic.RESNET50_NUMELS, [1], [127, 129, 1, 5000]):
        for p in (1, 2, 3, 4, 8):
            fmts = [fmts_all[i] for i in rng.integers(0, len(fmts_all), len(numels))]
            assert aps.layout_mixed(p, numels, fmts) == (orc.total_tiles(p, numels),
                                                        orc.packed_bytes_mixed(p, numels, fmts))
            assert aps.layout_mixed(p, numels, [(4, 3)] * len(numels)) == aps.layout(p, 4, 3, numels)
    hyb = synthetic.resnet50_hybrid_formats()
    assert aps.layout_mixed(8, synthetic.RESNET50_NUMELS, hyb) == (
        orc.total_tiles(8, synthetic.RESNET50_NUMELS), orc.packed_bytes_mixed(8, synthetic.RESNET50_NUMELS, hyb))


def test_ring_schedule_is_a_ring(aps):
    """At every step rank r receives exactly the chunk rank r-1 sends; after
    p-1 steps rank r holds chunk r, accumulated in order c+1, ..., c (A14)."""
    for p in (2, 3, 4, 5, 8):
        order = {c: [c] for c in range(p)}  # chunk -> ranks whose data it holds, in add order
        # before step 0 each rank's chunk c holds only its own data; track chunk on rank
        holds = {(r, c): [r] for r in range(p) for c in range(p)}
        for s in range(p - 1):
            new = dict(holds)
            for r in range(p):
                send_c, recv_c = aps.ring_step(p, r, s)
                prev = (r - 1) % p
                assert aps.ring_step(p, prev, s)[0] == recv_c
                new[(r, recv_c)] = holds[(prev, recv_c)] + [r]
            holds = new
        for r in range(p):
            assert holds[(r, r)] == [(r + j) % p for j in range(1, p + 1)]
        del order


def test_host_errors(aps):
    L = aps.load()
    h = ctypes.c_void_p()
    n = (ctypes.c_int64 * 2)(100, 5)
    assert L.aps_init(ctypes.byref(h), 1, 2, 1, 0, 2, n, None, None) == 2     # e = 1 rejected
    assert L.aps_init(ctypes.byref(h), 5, 24, 1, 0, 2, n, None, None) == 2
    assert L.aps_init(ctypes.byref(h), 5, 2, 2, 2, 2, n, None, None) == 1     # rank >= world
    bad = (ctypes.c_int64 * 2)(100, 0)
    assert L.aps_init(ctypes.byref(h), 5, 2, 1, 0, 2, bad, None, None) == 1
    assert L.aps_init(ctypes.byref(h), 5, 2, 1, 0, 2, n, None, None) == 0
    assert L.aps_workspace_bytes(h) > 16 * 8 * 2
    # no workspace yet: every device call is a state error, not a crash
    ptrs = (ctypes.c_void_p * 2)(16, 32)
    assert L.aps_layer_scales(h, ptrs) == 7
    assert L.aps_allreduce(h) == 7
    assert b"workspace" in L.aps_last_error(h)
    assert L.aps_destroy(h) == 0
    assert L.aps_ring_step(4, 4, 0, None, None) == 1
    assert L.aps_ring_step(4, 0, 3, None, None) == 1
