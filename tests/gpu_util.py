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
