"""NEXT-4 parity: sub-volume blocks extracted standalone and stitched (psn_block_gather ->
psn_extract -> psn_stitch_count / psn_stitch_scan / psn_stitch_emit) reproduce the whole-volume mesh
bit for bit -- against the oracle's whole-volume extraction (PAPER P:86-91 ids and order; P:264 open
boundaries; P:271 stitching) and against the CUDA path's own whole-volume psn_extract."""
import numpy as np
import pytest
import torch

import oracle
import gpu_util as gu

pytestmark = pytest.mark.gpu


def _blobs(rng, shape, dtype, nlab=5, noise=0.0):
    O, N, M = shape
    z, y, x = np.meshgrid(np.arange(O), np.arange(N), np.arange(M), indexing="ij")
    a = np.zeros(shape, np.int64)
    for lab in range(1, nlab + 1):
        c = rng.uniform(0, 1, 3) * np.array([M, N, O])
        r = rng.uniform(0.15, 0.45) * min(M, N, O)
        a[(x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 <= r * r] = lab
    if noise:
        m = rng.random(shape) < noise
        a[m] = rng.integers(0, nlab + 1, int(m.sum()))
    return a.astype(dtype)


def _stitched(a, blocks=None, cuts=None, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0), label_set=None,
              host=False, keep_local=True):
    from paper_2401_14906_b200.blocks import BlockedExtractor
    p = gu.psn()
    O, N, M = a.shape
    t = torch.from_numpy(np.ascontiguousarray(a))
    t = t.pin_memory() if host else t.cuda()
    bx = BlockedExtractor(p, (M, N, O), blocks=blocks or (1, 1, 1), cuts=cuts, spacing=spacing, origin=origin,
                          label_set=label_set, keep_local=keep_local)
    return bx.run(t), bx


def _assert_same(ms, a, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0), label_set=None, whole=True):
    om = oracle.extract(oracle.as_volume(a, spacing, origin, label_set))
    assert (ms.n_points, ms.n_quads, ms.n_stencil) == (om.n_points, om.n_quads, om.n_stencil)
    gu.assert_mesh_equal(gu.mesh_np(ms), om)
    if whole:   # and the CUDA whole-volume extraction (same bytes)
        _, _, mw, _ = gu.gpu_extract(a, spacing, origin, label_set)
        g, w = gu.mesh_np(ms), gu.mesh_np(mw)
        for k in g:
            np.testing.assert_array_equal(g[k], w[k], err_msg=k)
    return om


@pytest.mark.parametrize("blocks", [(1, 1, 1), (2, 1, 1), (1, 3, 1), (1, 1, 2), (2, 2, 2), (3, 2, 4)])
def test_blocks_bit_exact(blocks):
    rng = np.random.default_rng(271 + sum(blocks))
    a = _blobs(rng, (21, 26, 37), np.uint16, nlab=6, noise=0.02)
    ms, _ = _stitched(a, blocks=blocks, spacing=(0.8, 1.0, 1.5), origin=(-3.0, 2.0, 10.0))
    _assert_same(ms, a, (0.8, 1.0, 1.5), (-3.0, 2.0, 10.0))


def test_blocks_thin_and_ragged_cuts():
    """One-voxel blocks on every axis (the margin is the whole neighbour) and uneven cuts."""
    rng = np.random.default_rng(5)
    a = _blobs(rng, (13, 17, 19), np.uint8, nlab=4, noise=0.15)
    cuts = [[0, 1, 2, 9, 17, 18], [0, 1, 8, 15, 16], [0, 5, 6, 12]]
    ms, _ = _stitched(a, cuts=cuts)
    _assert_same(ms, a)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.uint32])
def test_blocks_dtypes_and_label_subset(dtype):
    rng = np.random.default_rng(11)
    a = _blobs(rng, (17, 15, 23), dtype, nlab=7, noise=0.05)
    if dtype == np.uint32:
        a = (a.astype(np.uint64) * 40000007 % (1 << 32)).astype(np.uint32)
        vals = np.unique(a)
        ls = [int(v) for v in vals[1::2]]
    else:
        ls = [1, 3, 4, 6]
    ms, _ = _stitched(a, blocks=(2, 2, 2), label_set=ls)
    _assert_same(ms, a, label_set=ls)


def test_blocks_out_of_core_host_volume():
    """Labels in pinned host memory, one block resident at a time (keep_local=False re-extracts)."""
    rng = np.random.default_rng(99)
    a = _blobs(rng, (30, 22, 41), np.uint16, nlab=9, noise=0.01)
    ms, _ = _stitched(a, blocks=(3, 2, 2), host=True, keep_local=False, spacing=(0.5, 0.7, 2.0))
    _assert_same(ms, a, (0.5, 0.7, 2.0))


def test_blocks_empty_and_iid():
    """Blocks without points (all background / one label) next to blocks with near-maximal output."""
    rng = np.random.default_rng(3)
    a = np.zeros((12, 14, 16), np.uint8)
    a[:, :, 8:] = rng.integers(0, 4, (12, 14, 8))
    ms, _ = _stitched(a, blocks=(2, 2, 2))
    _assert_same(ms, a)
    z = np.full((6, 7, 8), 3, np.uint8)
    ms, _ = _stitched(z, blocks=(2, 2, 2))
    assert (ms.n_points, ms.n_quads, ms.n_stencil) == (0, 0, 0)
    assert ms.stencil_offsets[:1].cpu().item() == 0


def test_blocks_smoothing_matches_whole():
    """The stitched mesh smooths like the whole-volume one (same CSR -> same Jacobi bits)."""
    rng = np.random.default_rng(8)
    a = _blobs(rng, (18, 20, 22), np.uint16, nlab=5)
    ms, bx = _stitched(a, blocks=(2, 2, 1), spacing=(0.8, 0.8, 1.5))
    p, vol, mw, _ = gu.gpu_extract(a, (0.8, 0.8, 1.5))
    ps = p.smooth(ms.volume, ms, 10, 0.5, 0.5)
    pw = p.smooth(vol, mw, 10, 0.5, 0.5)
    np.testing.assert_array_equal(ps[:ms.n_points].cpu().numpy(), pw[:mw.n_points].cpu().numpy())


def test_blocks_config_c2_full():
    """BASELINE c2 (256^3 u8, 20 Voronoi labels in an ellipsoid) in 2x2x2 blocks == whole volume."""
    import psn_gen
    a = psn_gen.generate_host(psn_gen.config("c2"))
    ms, _ = _stitched(a, blocks=(2, 2, 2))
    _, _, mw, _ = gu.gpu_extract(a)
    g, w = gu.mesh_np(ms), gu.mesh_np(mw)
    for k in g:
        np.testing.assert_array_equal(g[k], w[k], err_msg=k)


def test_blocks_config_c4_full():
    """BASELINE c4 (1024^3 u16) in 2x2x2 blocks, labels in pinned host memory, one block resident at a
    time: every stitched array == the whole-volume extraction's."""
    import psn_gen
    spec = psn_gen.config("c4")
    dev = psn_gen.generate_device(spec)
    p = gu.psn()
    mw = p.extract(p.volume(dev))
    w = gu.mesh_np(mw)
    host = dev.cpu().pin_memory()
    del dev, mw
    from paper_2401_14906_b200.blocks import BlockedExtractor
    M, N, O = spec.dims
    ms = BlockedExtractor(p, (M, N, O), blocks=(2, 2, 2), keep_local=False).run(host)
    g = gu.mesh_np(ms)
    for k in g:
        np.testing.assert_array_equal(g[k], w[k], err_msg=k)
