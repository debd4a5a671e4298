"""Peer (NVLink) halo push of the slab / shard smoothing loop,
on ONE GPU without ranks waiting on one another.

psn_smooth_step_peer stores a rank's boundary layers straight into its
neighbours' offset buffers and signals them; a step starts once both
neighbours finished the previous one.  Here every "rank" is a slab (or a
balanced shard) of one volume in this process, its peer pointers are simply
the other slabs' buffers on the same device, and the steps are launched rank by
rank, iteration by iteration, on one stream -- so when rank r runs iteration g,
its neighbours' iteration g-1 has already completed and no kernel waits on
another.  The concatenated result must equal the single-GPU psn_smooth bit for
bit.  The CUDA IPC export / open used across processes is tested separately
(two processes, one GPU, no kernel waiting)."""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest
import torch

import gpu_util as gu
import psn_gen
from paper_2401_14906_b200 import balance
from paper_2401_14906_b200.dist import peer_sides, shard_sends, slab_sends
from paper_2401_14906_b200.psn import Peer
from test_gpu_balance import extract_slabs
from test_gpu_slabs import concat

pytestmark = pytest.mark.gpu


def peer_loop(p, vols, meshes, sws, bufs, sends, G, T, lam, d):
    """T peer steps of G emulated ranks (sequential launches, one stream)."""
    sigs = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(G)]
    ctrs = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(G)]
    errs = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(G)]
    peers = []
    for r in range(G):
        lower, upper = peer_sides(r, G, sends)
        pr = Peer()
        pr.sig, pr.ctr, pr.err = sigs[r].data_ptr(), ctrs[r].data_ptr(), errs[r].data_ptr()
        for k, (nb, spec) in enumerate(((r - 1, lower), (r + 1, upper))):
            if spec is None:
                continue
            side = pr.side[k]
            side.dst[0], side.dst[1] = bufs[nb][0].data_ptr(), bufs[nb][1].data_ptr()
            side.src_begin, side.src_end, side.dst_begin = spec
            side.peer_sig = sigs[nb].data_ptr() + 8 * (1 - k)
        peers.append(pr)
    src = [None] * G
    for t in range(T):
        for r in range(G):
            p.smooth_step_peer(vols[r], meshes[r], sws[r], src[r], bufs[r][t & 1], t & 1, lam, d, peers[r])
        src = [bufs[r][t & 1] for r in range(G)]
    torch.cuda.synchronize()
    assert all(int(e.item()) == 0 for e in errs)
    # every rank signalled every iteration to each neighbour it exchanges with
    for r in range(G):
        lower, upper = peer_sides(r, G, sends)
        if lower is not None:
            assert int(sigs[r][0].item()) == T
        if upper is not None:
            assert int(sigs[r][1].item()) == T
        assert peers[r].iteration == T
    return src


def volume():
    rng = np.random.default_rng(7)
    a = np.zeros((26, 21, 37), np.uint16)
    a[1:-1, 1:-1, 1:-1] = rng.integers(0, 4, size=(24, 19, 35))
    z, y, x = np.meshgrid(np.arange(26), np.arange(21), np.arange(37), indexing="ij")
    a[((x - 18) ** 2 + (y - 10) ** 2 + (z - 12) ** 2) < 40] = 9
    return a


@pytest.mark.parametrize("G,shape,split", [(2, 0, 0), (3, 0, 0), (5, 0, 0), (3, 1, 0), (2, 0, 1), (3, 0, 1), (5, 0, 1),
                                           (3, 1, 1)])
def test_peer_slabs_match_single(monkeypatch, G, shape, split):
    """Peer-push slab smoothing equals one-GPU psn_smooth bit for bit -- with the 8-byte cache, and with the
    split cache psn_smooth_run_peer uses (split: step 0 writes it, steps 1.. read it; PSN_PEER_STEP_SPLIT)."""
    if split:
        monkeypatch.setenv("PSN_PEER_STEP_SPLIT", "1")
    p = gu.psn()
    p.set_constraint(shape)   # box, or the sphere (reading Q26)
    try:
        _peer_slabs_match_single(p, G)
    finally:
        p.set_constraint(0)


def _peer_slabs_match_single(p, G):
    a = volume()
    T, lam, d = 7, 0.5, 0.5
    vols, meshes, firsts, total = extract_slabs(p, a, G, (1.0, 1.0, 1.0))
    table = torch.tensor([[m.n_points, m.n_quads, m.n_stencil, m.c.halo_lo_points, m.c.halo_hi_points]
                          for m in meshes])
    sws = [p.smooth_workspace(m) for m in meshes]
    for r in range(G):
        p.smooth_prepare(vols[r], meshes[r], sws[r])
    bufs = [[p.offsets_buffer(m.n_window, "cuda") for _ in range(2)] for m in meshes]
    src = peer_loop(p, vols, meshes, sws, bufs, slab_sends(table), G, T, lam, d)
    outs = []
    for r in range(G):
        out = torch.empty((max(meshes[r].n_window, 1), 3), dtype=torch.float32, device="cuda")
        p.smooth_finalize(vols[r], meshes[r], src[r], out)
        outs.append(out)
    g = concat(meshes, outs)
    _, vol1, m1, _ = gu.gpu_extract(a)
    s1 = p.smooth(vol1, m1, T, lam, d)
    np.testing.assert_array_equal(g["smoothed"], s1[:m1.n_points].cpu().numpy())


@pytest.mark.parametrize("G,split", [(2, 0), (4, 0), (2, 1), (4, 1)])
def test_peer_balanced_shards_match_single(monkeypatch, G, split):
    if split:   # the split cache psn_smooth_run_peer uses, stepped rank by rank
        monkeypatch.setenv("PSN_PEER_STEP_SPLIT", "1")
    p = gu.psn()
    host = psn_gen.generate_host(psn_gen.config("c2"))[60:140]
    T, lam, d = 9, 0.5, 0.5
    vols, meshes, firsts, total = extract_slabs(p, host, G, (1.0, 1.0, 1.0))
    sources = [balance.source_from_mesh(m, f[0], f[1]) for m, f in zip(meshes, firsts)]
    cuts = balance.balanced_cuts(total, G)
    moves = balance.plan_moves([(s.first_point, s.n_points) for s in sources], cuts)
    shards = [balance.assemble_local(r, cuts, moves, sources, "cuda") for r in range(G)]
    windows = [(sh.w0, sh.w1) for sh in shards]
    hm = balance.halo_moves(cuts, windows)
    smeshes = [balance.shard_mesh(p, sh) for sh in shards]
    sws = [p.smooth_workspace(m) for m in smeshes]
    for m, w, sh in zip(smeshes, sws, shards):
        if sh.n_points:
            p.smooth_prepare(vols[0], m, w)
    bufs = [[p.offsets_buffer(sh.w1 - sh.w0, "cuda") for _ in range(2)] for sh in shards]
    src = peer_loop(p, [vols[0]] * G, smeshes, sws, bufs, shard_sends(hm, windows), G, T, lam, d)
    got = []
    for r in range(G):
        sh = shards[r]
        out = torch.empty((max(sh.w1 - sh.w0, 1), 3), dtype=torch.float32, device="cuda")
        p.smooth_finalize(vols[0], smeshes[r], src[r], out, sh.halo_lo, sh.halo_lo + sh.n_points)
        got.append(out[sh.halo_lo:sh.halo_lo + sh.n_points])
    got = torch.cat(got).cpu().numpy()
    _, vol1, m1, _ = gu.gpu_extract(host)
    s1 = p.smooth(vol1, m1, T, lam, d)
    np.testing.assert_array_equal(got, s1[:m1.n_points].cpu().numpy())


@pytest.mark.parametrize("G", [2, 3, 5])
def test_peer_point_balanced_slabs_match_single(G):
    """bench.py's default N > 1 partition: voxel-layer slabs cut to equal point counts
    (dist.balanced_layer_cuts on the per-layer counts from psn_extract_rows), extraction and peer
    smoothing on those uneven slabs == single-GPU psn_smooth bit for bit."""
    from paper_2401_14906_b200.dist import balanced_layer_cuts
    p = gu.psn()
    host = psn_gen.generate_host(psn_gen.config("c2"))[40:150]
    O, N, M = host.shape
    _, vol1, m1, _ = gu.gpu_extract(host)
    counts, _ = p.rows(vol1, m1.ws)
    layer_pts = counts[0].to(torch.int64).view(O - 1, N - 1).sum(1).tolist()
    parts = balanced_layer_cuts(layer_pts, G)
    assert parts != [(r * (O - 1) // G, (r + 1) * (O - 1) // G) for r in range(G)]   # really uneven
    T, lam, d = 6, 0.5, 0.5
    vols, meshes, firsts, total = extract_slabs(p, host, G, (1.0, 1.0, 1.0), parts=parts)
    pts_per_rank = [m.n_points for m in meshes]
    assert max(pts_per_rank) <= total / G + max(layer_pts)
    table = torch.tensor([[m.n_points, m.n_quads, m.n_stencil, m.c.halo_lo_points, m.c.halo_hi_points]
                          for m in meshes])
    sws = [p.smooth_workspace(m) for m in meshes]
    for r in range(G):
        p.smooth_prepare(vols[r], meshes[r], sws[r])
    bufs = [[p.offsets_buffer(m.n_window, "cuda") for _ in range(2)] for m in meshes]
    src = peer_loop(p, vols, meshes, sws, bufs, slab_sends(table), G, T, lam, d)
    outs = []
    for r in range(G):
        out = torch.empty((max(meshes[r].n_window, 1), 3), dtype=torch.float32, device="cuda")
        p.smooth_finalize(vols[r], meshes[r], src[r], out)
        outs.append(out)
    g = concat(meshes, outs)
    s1 = p.smooth(vol1, m1, T, lam, d)
    np.testing.assert_array_equal(g["smoothed"], s1[:m1.n_points].cpu().numpy())


def test_peer_slab_cut_above_flat_top_face():
    """A slab cut directly above an object's flat top face: rank 1's first own layer holds no
    points while rank 0's last one does, so rank 1 only RECEIVES on its lower side (peer_sides
    gives it the empty push (0, 0, 0) with a non-zero halo) -- accepted, signalled, bit-exact."""
    from paper_2401_14906_b200.dist import partition
    p = gu.psn()
    O, N, M = 20, 12, 14
    k0 = partition(O - 1, 2)[1][0]
    a = np.zeros((O, N, M), np.uint16)
    a[3:k0, 2:N - 2, 2:M - 3] = 3          # top face in lattice slice k0-1: voxel layer k0-1 has points, k0 none
    a[5:k0, 4:6, 4:6] = 5
    vols, meshes, firsts, total = extract_slabs(p, a, 2, (1.0, 1.0, 1.0))
    table = torch.tensor([[m.n_points, m.n_quads, m.n_stencil, m.c.halo_lo_points, m.c.halo_hi_points]
                          for m in meshes])
    assert meshes[1].c.halo_lo_points > 0
    sends = slab_sends(table)
    lower, _ = peer_sides(1, 2, sends)
    assert lower is not None and lower[1] <= lower[0]     # rank 1 pushes nothing down
    T, lam, d = 5, 0.5, 0.5
    sws = [p.smooth_workspace(m) for m in meshes]
    for r in range(2):
        p.smooth_prepare(vols[r], meshes[r], sws[r])
    bufs = [[p.offsets_buffer(m.n_window, "cuda") for _ in range(2)] for m in meshes]
    src = peer_loop(p, vols, meshes, sws, bufs, sends, 2, T, lam, d)
    outs = []
    for r in range(2):
        out = torch.empty((max(meshes[r].n_window, 1), 3), dtype=torch.float32, device="cuda")
        p.smooth_finalize(vols[r], meshes[r], src[r], out)
        outs.append(out)
    g = concat(meshes, outs)
    _, vol1, m1, _ = gu.gpu_extract(a)
    s1 = p.smooth(vol1, m1, T, lam, d)
    np.testing.assert_array_equal(g["smoothed"], s1[:m1.n_points].cpu().numpy())


def test_peer_step_argument_errors():
    from paper_2401_14906_b200.psn import PSNError, PSN_ERR_ARG
    p = gu.psn()
    a = volume()
    vols, meshes, firsts, total = extract_slabs(p, a, 2, (1.0, 1.0, 1.0))
    ws = p.smooth_workspace(meshes[0])
    p.smooth_prepare(vols[0], meshes[0], ws)
    dst = p.offsets_buffer(meshes[0].n_window, "cuda")
    pr = Peer()
    with pytest.raises(PSNError) as e:   # no signal / counter words
        p.smooth_step_peer(vols[0], meshes[0], ws, None, dst, 0, 0.5, 0.5, pr)
    assert e.value.status == PSN_ERR_ARG
    sig = torch.zeros(2, dtype=torch.int64, device="cuda")
    ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    pr.sig, pr.ctr, pr.err = sig.data_ptr(), ctr.data_ptr(), err.data_ptr()
    other = p.offsets_buffer(meshes[1].n_window, "cuda")
    pr.side[1].dst[0] = pr.side[1].dst[1] = other.data_ptr()
    pr.side[1].peer_sig = sig.data_ptr()
    pr.side[1].src_begin, pr.side[1].src_end = 0, meshes[0].n_window + 1   # beyond the own entries
    with pytest.raises(PSNError) as e:
        p.smooth_step_peer(vols[0], meshes[0], ws, None, dst, 0, 0.5, 0.5, pr)
    assert e.value.status == PSN_ERR_ARG
    with pytest.raises(PSNError) as e:
        p.smooth_step_peer(vols[0], meshes[0], ws, None, dst, 2, 0.5, 0.5, pr)
    assert e.value.status == PSN_ERR_ARG


class _CudaArray:
    """A raw device pointer as a torch-importable array (__cuda_array_interface__)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 2}


def _ipc_child(q_in, q_out):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2401_14906_b200 import PSN
    p = PSN(0)
    blob, n = q_in.get()
    addr = p.ipc_open(blob)
    t = torch.as_tensor(_CudaArray(addr, n), device="cuda")
    t.copy_(torch.arange(n, dtype=torch.float32, device="cuda") * 2.0 + 1.0)
    torch.cuda.synchronize()
    p.ipc_close(addr)
    q_out.put("done")


def test_ipc_export_open_across_processes():
    """Process B maps process A's exported sub-allocation (non-zero offset inside a
    cudaMalloc block) and writes it; A sees the values.  One GPU, no kernel waits."""
    p = gu.psn()
    big = torch.zeros(1 << 20, dtype=torch.float32, device="cuda")
    view = big[4096:4096 + 1000]   # offset inside the allocation
    blob = p.ipc_export(view)
    ctx = mp.get_context("spawn")
    q_in, q_out = ctx.Queue(), ctx.Queue()
    proc = ctx.Process(target=_ipc_child, args=(q_in, q_out))
    proc.start()
    q_in.put((blob, 1000))
    assert q_out.get(timeout=120) == "done"
    proc.join(timeout=60)
    assert proc.exitcode == 0
    torch.cuda.synchronize()
    np.testing.assert_array_equal(view.cpu().numpy(), np.arange(1000, dtype=np.float32) * 2.0 + 1.0)
    assert float(big[:4096].abs().sum()) == 0.0 and float(big[5096:].abs().sum()) == 0.0


def test_run_peer_single_rank_matches_single():
    """psn_smooth_run_peer (all steps in one call) on a rank without neighbours equals
    psn_smooth bit for bit (the multi-rank interleaving is covered step by step above:
    in one process a rank's later steps would wait on the others)."""
    p = gu.psn()
    a = volume()
    T, lam, d = 8, 0.5, 0.5
    vols, meshes, firsts, total = extract_slabs(p, a, 1, (1.0, 1.0, 1.0))
    ws = p.smooth_workspace(meshes[0])
    p.smooth_prepare(vols[0], meshes[0], ws)
    bufs = [p.offsets_buffer(meshes[0].n_window, "cuda") for _ in range(2)]
    sig = torch.zeros(2, dtype=torch.int64, device="cuda")
    ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    pr = Peer()
    pr.sig, pr.ctr, pr.err = sig.data_ptr(), ctr.data_ptr(), err.data_ptr()
    _, vol1, m1, _ = gu.gpu_extract(a)
    s1 = p.smooth(vol1, m1, T, lam, d)
    # two runs back to back (T odd the second time): the buffer parity continues from the global
    # iteration, and each run's result (in bufs[(iteration - 1) & 1]) equals psn_smooth
    for run, TT in enumerate((T, T - 1)):
        s1 = p.smooth(vol1, m1, TT, lam, d)
        g0 = pr.iteration
        res = p.smooth_run_peer(vols[0], meshes[0], ws, bufs, TT, lam, d, pr)
        assert res is bufs[(g0 + TT - 1) & 1]
        out = torch.empty((meshes[0].n_window, 3), dtype=torch.float32, device="cuda")
        p.smooth_finalize(vols[0], meshes[0], res, out)
        np.testing.assert_array_equal(out[:m1.n_points].cpu().numpy(), s1[:m1.n_points].cpu().numpy())
    assert pr.iteration == 2 * T - 1 and int(err.item()) == 0
