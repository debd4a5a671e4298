"""The peer halo push across PROCESSES (dist.PeerHalo: CUDA IPC export / open,
all-gathered handles, psn_smooth_step_peer), two ranks on ONE GPU.

The ranks are separate processes (gloo for the host-side all-gathers) sharing
cuda:0.  They step in lockstep -- every step is followed by a device sync and a
barrier -- so when a rank launches step g its neighbour's step g-1 has already
completed: no kernel ever waits on another (what a multi-GPU run overlaps is
serialised here).  The concatenated smoothed points must equal the single-GPU
psn_smooth bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _volume():
    rng = np.random.default_rng(11)
    a = np.zeros((22, 19, 33), np.uint16)
    a[1:-1, 1:-1, 1:-1] = rng.integers(0, 4, size=(20, 17, 31))
    return a


def _worker(rank, world, port, T, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    from paper_2401_14906_b200 import PSN
    from paper_2401_14906_b200.dist import PeerHalo, peer_sides, slab_sends
    from test_gpu_balance import extract_slabs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        p = PSN(0)
        a = _volume()
        vols, meshes, firsts, total = extract_slabs(p, a, world, (1.0, 1.0, 1.0))   # every slab (cheap)
        table = torch.tensor([[m.n_points, m.n_quads, m.n_stencil, m.c.halo_lo_points, m.c.halo_hi_points]
                              for m in meshes])
        vol, mesh = vols[rank], meshes[rank]
        ws = p.smooth_workspace(mesh)
        p.smooth_prepare(vol, mesh, ws)
        bufs = [p.offsets_buffer(mesh.n_window, "cuda") for _ in range(2)]
        lower, upper = peer_sides(rank, world, slab_sends(table))
        ph = PeerHalo(p, bufs, lower, upper, group=None)
        src = None
        for t in range(T):
            ph.step(vol, mesh, ws, src, bufs[t & 1], t & 1, 0.5, 0.5)
            src = bufs[t & 1]
            torch.cuda.synchronize()
            dist.barrier()   # lockstep: the neighbour's step t is complete before anyone launches t + 1
        ph.check()
        out = torch.empty((mesh.n_window, 3), dtype=torch.float32, device="cuda")
        p.smooth_finalize(vol, mesh, src, out)
        torch.cuda.synchronize()
        hl = mesh.c.halo_lo_points
        mine = out[hl:hl + mesh.n_points].cpu().numpy()
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        dist.barrier()
        ph.close()
        if rank == 0:
            q.put(np.concatenate(allp))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_peer_halo_two_processes_one_gpu():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import gpu_util as gu
    T, world = 6, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    p = gu.psn()
    a = _volume()
    _, vol1, m1, _ = gu.gpu_extract(a)
    ref = p.smooth(vol1, m1, T, 0.5, 0.5)[:m1.n_points].cpu().numpy()
    np.testing.assert_array_equal(got, ref)


def _layer_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    from paper_2401_14906_b200 import PSN
    from paper_2401_14906_b200.dist import balanced_layer_cuts, gather_layer_points, partition, slab_slices
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        p = PSN(0)
        a = _volume()
        O, N, M = a.shape
        own = partition(O - 1, world)[rank]
        z_lo, z_hi = slab_slices(O, own[0], own[1])
        dev = torch.from_numpy(np.ascontiguousarray(a[z_lo:z_hi])).cuda()
        vol = p.volume(dev, dims=(M, N, O), z_lo=z_lo, own=own)
        ws = p.workspace(vol)
        p.count(vol, p.labels(None), ws)
        pts = gather_layer_points(p, vol, ws, own)
        if rank == 0:
            q.put((pts, balanced_layer_cuts(pts, world)))
    finally:
        dist.destroy_process_group()


def test_gather_layer_points_two_processes():
    """bench.py's N > 1 partition step across processes: every rank's per-layer point counts (from
    psn_extract_rows on its slab) all-gathered into the whole volume's list == the single-volume
    per-layer counts, and the balanced cuts computed from them."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import gpu_util as gu
    from paper_2401_14906_b200.dist import balanced_layer_cuts
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_layer_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    pts, cuts = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    p = gu.psn()
    a = _volume()
    O, N, M = a.shape
    _, vol1, m1, _ = gu.gpu_extract(a)
    counts, _ = p.rows(vol1, m1.ws)
    ref = counts[0].to(torch.int64).view(O - 1, N - 1).sum(1).tolist()
    assert pts == ref
    assert cuts == balanced_layer_cuts(ref, world)
