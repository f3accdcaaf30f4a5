"""CPU checks of the product library: it loads, exports every symbol that
include/mrf_cuda.h declares, rejects invalid arguments like the reference, and
its host-side topology (scanline order, edge numbering, dir offsets -- the p/q
byte layout) is identical to the reference's for every small grid and all 16
directions (acceptance.cpp:297-325 partition, test_grid.cpp:110-134)."""
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_1910_10892_b200 import _lib
from paper_1910_10892_b200.api import GridTopology

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "mrf_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mrf_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.mrf_version() == 20000  # MRF_VERSION in include/mrf_cuda.h


def test_invalid_arguments_rejected():
    import ctypes as C

    h = C.c_void_p()
    assert _lib.lib().mrf_topology_create(4, 4, 6, C.byref(h)) == _lib.MRF_EINVAL
    assert b"connectivity" in _lib.lib().mrf_last_error()
    assert _lib.lib().mrf_topology_create(0, 4, 4, C.byref(h)) == _lib.MRF_EINVAL
    with pytest.raises(ValueError):
        GridTopology(3, 3, 5)


@pytest.mark.parametrize("conn", [4, 8, 16])
def test_topology_matches_restatement_all_small_grids(conn):
    for H in range(1, 17):
        for W in range(1, 17):
            t = GridTopology(H, W, conn)
            o = O.oracle_topology(H, W, conn)
            assert t.total_edges == o.total_edges
            assert np.array_equal(t.dir_offset, o.dir_offset)
            assert np.array_equal(t.edge_index(), o.edge_index), (H, W)
            for r in range(conn):
                first, length = t.scanlines(r)
                assert np.array_equal(first, o.line_first[r]), (H, W, r)
                assert np.array_equal(length, o.line_len[r]), (H, W, r)


@pytest.mark.skipif(not O.have_ref(), reason="reference library not built here")
@pytest.mark.parametrize("H,W", [(375, 1242), (288, 384), (500, 750), (33, 17), (1, 40), (40, 1)])
def test_topology_matches_reference_config_shapes(H, W):
    for conn in (4, 8, 16):
        t = GridTopology(H, W, conn)
        r_ = O.ref_topology(H, W, conn)
        assert t.total_edges == r_.total_edges
        assert np.array_equal(t.edge_index(), r_.edge_index)
        for r in range(conn):
            first, length = t.scanlines(r)
            assert np.array_equal(first, r_.line_first[r]) and np.array_equal(length, r_.line_len[r])


def test_index_footprint_formula():
    """IndexStore::bytes() = K * sum_r |E^r| * (L+1) with |E^r| = (H-|dh|)(W-|dw|)."""
    for (H, W, conn) in [(5, 8, 4), (5, 8, 8), (6, 6, 16), (375, 1242, 4), (500, 750, 8)]:
        t = GridTopology(H, W, conn)
        steps = [(0, 1), (0, -1), (1, 0), (-1, 0), (1, 1), (-1, -1), (1, -1), (-1, 1),
                 (1, 2), (-1, -2), (1, -2), (-1, 2), (2, 1), (-2, -1), (2, -1), (-2, 1)][:conn]
        E = sum(max(0, H - abs(a)) * max(0, W - abs(b)) for a, b in steps)
        assert t.total_edges == E
        assert t.index_bytes(7, 3) == 3 * E * 8
