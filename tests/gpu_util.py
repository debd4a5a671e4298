"""Helpers for the -m gpu parity tests: run the CUDA path through the C ABI
(paper_2401_14906_b200.PSN) and the oracle on the same bytes, and compare."""
import numpy as np
import torch

import oracle

_psn = None


def psn():
    global _psn
    if _psn is None:
        from paper_2401_14906_b200 import PSN
        _psn = PSN(0)
    return _psn


def u32(t, n):
    return t[:n].cpu().numpy().view(np.uint32) if n else np.zeros((0,) + tuple(t.shape[1:]), np.uint32)


def gpu_extract(labels_np, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0), label_set=None):
    p = psn()
    dev = torch.from_numpy(np.ascontiguousarray(labels_np)).cuda()
    vol = p.volume(dev, spacing=spacing, origin=origin)
    mesh = p.extract(vol, label_set)
    return p, vol, mesh, dev


def mesh_np(mesh):
    P, Q, S = mesh.n_points, mesh.n_quads, mesh.n_stencil
    nw = mesh.n_window
    return dict(points=mesh.points[:nw].cpu().numpy() if nw else np.zeros((0, 3), np.float32),
                quads=u32(mesh.quads, Q), pairs=u32(mesh.pairs, Q),
                csr_off=mesh.stencil_offsets[:P + 1].cpu().numpy().view(np.uint32),
                csr_ids=u32(mesh.stencil_ids, S),
                face_mask=mesh.face_masks[:P].cpu().numpy() if P else np.zeros(0, np.uint8))


def assert_mesh_equal(g, om, window_lo=0):
    """Bit-exact comparison of a GPU mesh (numpy dict) with an oracle Mesh."""
    P = om.n_points
    np.testing.assert_array_equal(g["points"][window_lo:window_lo + P], om.points)
    np.testing.assert_array_equal(g["quads"], om.quads)
    np.testing.assert_array_equal(g["pairs"], om.pairs)
    np.testing.assert_array_equal(g["csr_off"], om.csr_off)
    np.testing.assert_array_equal(g["csr_ids"], om.csr_ids)
    np.testing.assert_array_equal(g["face_mask"], om.face_mask)


def oracle_rows(om, dims, k0=0, k1=None):
    """Per voxel row (layers [k0, k1), r = j + (N-1)(k - k0)) of an oracle mesh: P/Q/S counts and the
    tight point range [min i, max i + 1) ([0, 0) without points)."""
    M, N, O = dims
    k1 = O - 1 if k1 is None else k1
    R = (N - 1) * (k1 - k0)
    vi = om.voxel_idx
    r = vi[:, 1] + (N - 1) * (vi[:, 2] - k0)
    deg = np.diff(om.csr_off.astype(np.int64))
    P = np.bincount(r, minlength=R)
    Q = np.bincount(r[om.quads[:, 2].astype(np.int64) - om.point_base], minlength=R) if om.n_quads else np.zeros(R, np.int64)
    S = np.bincount(r, weights=deg, minlength=R).astype(np.int64)
    lo = np.zeros(R, np.int64); hi = np.zeros(R, np.int64)
    if om.n_points:
        starts = np.flatnonzero(np.r_[True, r[1:] != r[:-1]])
        rows = r[starts]
        lo[rows] = np.minimum.reduceat(vi[:, 0], starts)
        hi[rows] = np.maximum.reduceat(vi[:, 0], starts) + 1
    return np.stack([P, Q, S]), np.stack([lo, hi], -1)


def check_rows(g_counts, g_trims, om, ovol, k0=0, k1=None):
    """S:602 planned per-row counts == emitted per-row counts (the oracle's), and the GPU's trims
    are the tight point ranges, inside the paper's voxel-row range from the oracle's Pass-2 grid-row
    trims ([max(0, minL-1), min(maxR, M-1)) over grid rows (j..j+1, k..k+1))."""
    M, N, O = ovol.dims
    k1 = O - 1 if k1 is None else k1
    cnt, tr = oracle_rows(om, ovol.dims, k0, k1)
    np.testing.assert_array_equal(g_counts.astype(np.int64), cnt)
    np.testing.assert_array_equal(g_trims.astype(np.int64), tr)
    _, fin = oracle.row_trims(ovol, k0, k1 + 1)            # grid rows of slices [k0, k1]
    has = fin[..., 1] > fin[..., 0]
    big = np.iinfo(np.int64).max
    lo4 = np.where(has, fin[..., 0], big)
    hi4 = np.where(has, fin[..., 1], -1)
    minL = np.minimum.reduce([lo4[:-1, :-1], lo4[:-1, 1:], lo4[1:, :-1], lo4[1:, 1:]]).reshape(-1)
    maxR = np.maximum.reduce([hi4[:-1, :-1], hi4[:-1, 1:], hi4[1:, :-1], hi4[1:, 1:]]).reshape(-1)
    pts = cnt[0] > 0
    assert np.all(tr[pts, 0] >= np.maximum(0, minL[pts] - 1))
    assert np.all(tr[pts, 1] <= np.minimum(maxR[pts], M - 1))
