"""CPU checks of the C-ABI boundary: libpsn.so loads without a GPU and exports every function
include/psn.h declares (and the binding's list matches); the host-only entry points (workspace
sizes, psn_block_box, status strings) behave as documented.  No compute call needs a GPU here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "psn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(psn_\w+)\s*\(", src, flags=re.M)))


def _lib():
    from paper_2401_14906_b200 import psn as P
    if not os.path.exists(P.LIB_PATH):
        pytest.skip("libpsn.so not built")
    return P, P.lib()


def test_header_symbols_exported():
    P, L = _lib()
    names = _declared()
    assert len(names) >= 30, names
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(P.EXPORTED) == names


def test_status_strings():
    _, L = _lib()
    for s in range(7):
        assert L.psn_status_string(s)


def test_block_box_margins():
    P, L = _lib()
    b = P.Block()
    dims = (20, 15, 9)
    for a in range(3):
        b.dims[a] = dims[a]
    own = [(0, 7), (5, 14), (3, 4)]
    for a in range(3):
        b.own_lo[a], b.own_hi[a] = own[a]
    b.xseg, b.nxseg = 0, 2
    assert L.psn_block_box(ctypes.byref(b), 0) == P.PSN_OK
    # interior sides get one margin voxel (lattice lo-1 .. hi+1), volume sides none
    assert [b.box_lo[a] for a in range(3)] == [0, 4, 2]
    assert [b.box_hi[a] for a in range(3)] == [9, 15, 6]
    # 16-byte rows: u16 -> x width a multiple of 8 (grown on the right inside M = 20)
    assert L.psn_block_box(ctypes.byref(b), 2) == P.PSN_OK
    assert (b.box_lo[0], b.box_hi[0]) == (0, 16)
    # last x-block: grown to the left
    b.own_lo[0], b.own_hi[0], b.xseg = 7, 19, 1
    assert L.psn_block_box(ctypes.byref(b), 2) == P.PSN_OK
    assert (b.box_lo[0], b.box_hi[0]) == (4, 20)
    assert L.psn_block_box(ctypes.byref(b), 1) == P.PSN_OK   # 16 u8 elements
    assert (b.box_lo[0], b.box_hi[0]) == (4, 20)
    assert L.psn_block_box(ctypes.byref(b), 3) == P.PSN_ERR_ARG
    b.own_lo[0], b.own_hi[0], b.xseg = 0, 7, 0
    assert L.psn_block_box(ctypes.byref(b), 0) == P.PSN_OK
    n = ctypes.c_size_t()
    assert L.psn_stitch_workspace(ctypes.byref(b), ctypes.byref(n)) == P.PSN_OK
    assert n.value >= 4 * 4 * (15 - 4 - 1) * (6 - 2 - 1)
    # inconsistent x-block index / empty box / outside the voxels
    b.xseg = 1
    assert L.psn_block_box(ctypes.byref(b), 0) == P.PSN_ERR_ARG
    b.xseg = 0
    b.own_hi[2] = 3
    assert L.psn_block_box(ctypes.byref(b), 0) == P.PSN_ERR_ARG
    b.own_hi[2] = 9
    assert L.psn_block_box(ctypes.byref(b), 0) == P.PSN_ERR_ARG


def test_scan_workspace_size():
    _, L = _lib()
    assert L.psn_stitch_scan_workspace(1) == 3 * 8
    assert L.psn_stitch_scan_workspace(4096 * 5 + 1) == 3 * 8 * 6


def test_block_cuts():
    from paper_2401_14906_b200.blocks import block_cuts
    for n in (1, 2, 7, 255, 1023):
        for p in (1, 2, 3, 8, 2000):
            c = block_cuts(n, p)
            assert c[0] == 0 and c[-1] == n and len(c) == min(p, n) + 1
            assert all(c[t] < c[t + 1] for t in range(len(c) - 1))
            sizes = [c[t + 1] - c[t] for t in range(len(c) - 1)]
            assert max(sizes) - min(sizes) <= 1


def test_block_grid_covers_voxels_once():
    """BlockedExtractor's grid (host logic, no GPU): every voxel owned by exactly one block, every box
    contains its own box plus the one-voxel margin on interior sides, x-block indices consistent."""
    import numpy as np
    P, L = _lib()
    from paper_2401_14906_b200.blocks import BlockedExtractor

    class Stub:
        pass
    s = Stub()
    s.L = L

    def check(rc):
        assert rc == P.PSN_OK
    s._check = check
    dims = (23, 17, 12)
    bx = BlockedExtractor(s, dims, blocks=(3, 2, 4))
    own = np.zeros((dims[2] - 1, dims[1] - 1, dims[0] - 1), np.int32)
    for b in bx.blocks:
        lo = [b.own_lo[a] for a in range(3)]; hi = [b.own_hi[a] for a in range(3)]
        own[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] += 1
        for a in range(3):
            assert b.box_lo[a] == max(lo[a] - 1, 0) and b.box_hi[a] == min(hi[a] + 2, dims[a])
        assert (b.xseg > 0) == (lo[0] > 0) and (b.xseg < b.nxseg - 1) == (hi[0] < dims[0] - 1)
    assert own.min() == 1 and own.max() == 1
    assert bx.nseg == (dims[1] - 1) * (dims[2] - 1) * 3
    with pytest.raises(ValueError):
        BlockedExtractor(s, dims, cuts=[[0, 5, 5, 22], [0, 16], [0, 11]])
