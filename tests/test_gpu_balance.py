"""Point-balanced smoothing re-partition, emulated on ONE GPU.

Each z-slab is extracted through psn_extract (equal slabs, one-slice halos),
then the smoothing ownership is re-cut into equal global-id ranges
(paper_2401_14906_b200.balance): every rank receives the face masks, CSR rows
and anchors of its new range from their extraction owners, smooths its shard
through psn_smooth_prepare / psn_smooth_step with the halo exchange of the new
windows (device copies standing in for NCCL), and finalizes its own ids.  The
concatenation in rank order must equal the single-GPU smoothing bit for bit and
match the oracle within 1e-4 * s."""
import numpy as np
import pytest
import torch

import gpu_util as gu
import oracle
import psn_gen
from paper_2401_14906_b200 import balance
from paper_2401_14906_b200.dist import partition, slab_slices

pytestmark = pytest.mark.gpu


def extract_slabs(p, a, G, spacing, parts=None):
    O, N, M = a.shape
    vols, counted, wss = [], [], []
    for (k0, k1) in (parts if parts is not None else partition(O - 1, G)):
        z_lo, z_hi = slab_slices(O, k0, k1)
        dev = torch.from_numpy(np.ascontiguousarray(a[z_lo:z_hi])).cuda()
        vol = p.volume(dev, dims=(M, N, O), spacing=spacing, z_lo=z_lo, own=(k0, k1))
        vol._keep = dev
        ws = p.workspace(vol)
        c = p.count(vol, p.labels(None), ws)
        vols.append(vol); counted.append(c); wss.append(ws)
    firsts, meshes = [], []
    fp = fq = fs = 0
    for r in range(G):
        meshes.append(p.emit(vols[r], p.labels(None), wss[r], counted[r], first=(fp, fq, fs)))
        firsts.append((fp, fs))
        fp += counted[r].n_points; fq += counted[r].n_quads; fs += counted[r].n_stencil
    return vols, meshes, firsts, fp


def smooth_balanced(p, vols, meshes, firsts, total, G, T, lam, d):
    sources = [balance.source_from_mesh(m, f[0], f[1]) for m, f in zip(meshes, firsts)]
    cuts = balance.balanced_cuts(total, G)
    moves = balance.plan_moves([(s.first_point, s.n_points) for s in sources], cuts)
    shards = [balance.assemble_local(r, cuts, moves, sources, "cuda") for r in range(G)]
    hm = balance.halo_moves(cuts, [(sh.w0, sh.w1) for sh in shards])
    smeshes = [balance.shard_mesh(p, sh) for sh in shards]
    sws = [p.smooth_workspace(m) for m in smeshes]
    for m, w in zip(smeshes, sws):
        p.smooth_prepare(vols[0], m, w)
    bufs = [[p.offsets_buffer(sh.w1 - sh.w0, "cuda") for _ in range(2)] for sh in shards]   # float4 offsets
    src = [None] * G
    for t in range(T):
        for r in range(G):
            if shards[r].n_points:
                p.smooth_step(vols[0], smeshes[r], sws[r], src[r], bufs[r][t & 1], lam, d)
        for (s, dd, g0, g1) in hm:   # halo exchange of the new windows
            bufs[dd][t & 1][g0 - shards[dd].w0:g1 - shards[dd].w0] = bufs[s][t & 1][g0 - shards[s].w0:g1 - shards[s].w0]
        src = [bufs[r][t & 1] for r in range(G)]
    outs = []
    for r in range(G):
        sh = shards[r]
        out = torch.empty((max(sh.w1 - sh.w0, 1), 3), dtype=torch.float32, device="cuda")
        if sh.n_points:
            p.smooth_finalize(vols[0], smeshes[r], src[r], out, sh.halo_lo, sh.halo_lo + sh.n_points)
        outs.append(out[sh.halo_lo:sh.halo_lo + sh.n_points])
    torch.cuda.synchronize()
    return torch.cat(outs).cpu().numpy(), shards, moves


@pytest.mark.parametrize("G", [2, 3, 5])
def test_balanced_smoothing_matches_single(G):
    rng = np.random.default_rng(300 + G)
    a = np.zeros((31, 22, 29), np.uint16)
    # surfaces concentrated in the lower layers: equal z-slabs are unbalanced in points
    a[1:12, 1:-1, 1:-1] = rng.integers(0, 4, size=(11, 20, 27))
    z, y, x = np.meshgrid(np.arange(31), np.arange(22), np.arange(29), indexing="ij")
    a[((x - 14) ** 2 + (y - 10) ** 2 + (z - 22) ** 2) < 20] = 7
    sp = (0.8, 1.0, 1.5)
    T, lam, d = 7, 0.5, 0.5
    p = gu.psn()
    vols, meshes, firsts, total = extract_slabs(p, a, G, sp)
    got, shards, moves = smooth_balanced(p, vols, meshes, firsts, total, G, T, lam, d)
    sizes = [sh.n_points for sh in shards]
    assert max(sizes) - min(sizes) <= 1                      # equal shares of the points
    assert any(src != dst for src, dst, _, _ in moves)      # the re-partition really moved points
    _, vol1, m1, _ = gu.gpu_extract(a, spacing=sp)
    ref_gpu = p.smooth(vol1, m1, T, lam, d)[:m1.n_points].cpu().numpy()
    np.testing.assert_array_equal(got, ref_gpu)
    om = oracle.extract(oracle.as_volume(a, sp))
    ref = oracle.smooth(om, sp, T, lam, d)
    assert (np.abs(got.astype(np.float64) - ref) / np.array(sp)).max() <= 1e-4


def test_balanced_smoothing_c2():
    host = psn_gen.generate_host(psn_gen.config("c2"))
    p = gu.psn()
    vols, meshes, firsts, total = extract_slabs(p, host, 4, (1.0, 1.0, 1.0))
    got, shards, _ = smooth_balanced(p, vols, meshes, firsts, total, 4, 25, 0.5, 0.5)
    _, vol1, m1, _ = gu.gpu_extract(host)
    np.testing.assert_array_equal(got, p.smooth(vol1, m1, 25, 0.5, 0.5)[:m1.n_points].cpu().numpy())
