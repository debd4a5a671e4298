"""Point-balanced smoothing re-partition (paper_2401_14906_b200.balance):
host planning on CPU, and the distributed re-partition + halo exchange over
gloo (world 2 and 3) on an oracle mesh split into equal z-slabs.  The GPU
smoothing on the shards is tested in tests/test_gpu_balance.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2401_14906_b200 import balance
from paper_2401_14906_b200.dist import assemble_batched, partition, p2p_transport, shard_halo_exchange


def test_cuts_and_moves_cover_ranges():
    for total, G in [(0, 3), (1, 4), (10, 3), (1_000_003, 8)]:
        cuts = balance.balanced_cuts(total, G)
        assert cuts[0] == 0 and cuts[-1] == total and all(b - a in (total // G, total // G + 1)
                                                           for a, b in zip(cuts, cuts[1:]))
    owned = [(0, 10), (10, 0), (10, 25), (35, 5)]
    cuts = balance.balanced_cuts(40, 4)
    moves = balance.plan_moves(owned, cuts)
    for dst in range(4):
        got = sorted((g0, g1) for s, d, g0, g1 in moves if d == dst)
        assert got[0][0] == cuts[dst] and got[-1][1] == cuts[dst + 1]
        assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
    for s, d, g0, g1 in moves:
        assert owned[s][0] <= g0 < g1 <= owned[s][0] + owned[s][1]


def test_halo_moves():
    cuts = [0, 10, 20, 30]
    windows = [(0, 13), (7, 24), (18, 30)]
    hm = balance.halo_moves(cuts, windows)
    assert sorted(hm) == sorted([(1, 0, 10, 13), (0, 1, 7, 10), (2, 1, 20, 24), (1, 2, 18, 20)])


def _mesh_and_slabs(G):
    rng = np.random.default_rng(7)
    a = np.zeros((17, 11, 13), np.uint8)
    a[1:8, 1:-1, 1:-1] = rng.integers(0, 3, size=(7, 9, 11))
    m = oracle.extract(oracle.as_volume(a))
    k = m.voxel_idx[:, 2]
    owned = []
    for (k0, k1) in partition(a.shape[0] - 1, G):
        ids = np.nonzero((k >= k0) & (k < k1))[0]
        owned.append((int(ids[0]) if len(ids) else int(np.searchsorted(k, k0)), len(ids)))
    return m, owned


def _source(m, f, n):
    off = m.csr_off[f:f + n + 1]
    return balance.SourceMesh(first_point=f, n_points=n, halo_lo=0, first_stencil=int(off[0]),
                              points=torch.from_numpy(m.points[f:f + n].copy()),
                              face_masks=torch.from_numpy(m.face_mask[f:f + n].copy()),
                              stencil_offsets=torch.from_numpy(off.astype(np.uint32).view(np.int32).copy()),
                              stencil_ids=torch.from_numpy(m.csr_ids[off[0]:off[-1]].astype(np.uint32).view(np.int32).copy()))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, owned = _mesh_and_slabs(world)
        cuts = balance.balanced_cuts(m.n_points, world)
        moves = balance.plan_moves(owned, cuts)
        src = _source(m, *owned[rank])
        sh = balance.assemble(rank, cuts, moves, src, p2p_transport(), "cpu")
        shb = assemble_batched(rank, cuts, moves, src, "cpu")   # the two-batch form BalancedSmoother uses
        assert (shb.a0, shb.a1, shb.w0, shb.w1) == (sh.a0, sh.a1, sh.w0, sh.w1)
        for key in ("face_masks", "stencil_offsets", "stencil_ids", "points"):
            assert torch.equal(getattr(shb, key), getattr(sh, key)), key
        a0, a1 = cuts[rank], cuts[rank + 1]
        assert (sh.a0, sh.a1) == (a0, a1)
        np.testing.assert_array_equal(sh.face_masks.numpy(), m.face_mask[a0:a1])
        np.testing.assert_array_equal(sh.stencil_offsets.numpy().view(np.uint32), m.csr_off[a0:a1 + 1])
        ids = m.csr_ids[m.csr_off[a0]:m.csr_off[a1]]
        np.testing.assert_array_equal(sh.stencil_ids.numpy().view(np.uint32), ids)
        np.testing.assert_array_equal(sh.points[sh.halo_lo:sh.halo_lo + sh.n_points].numpy(), m.points[a0:a1])
        assert sh.w0 == min(a0, int(ids.min()) if len(ids) else a0)
        assert sh.w1 == max(a1, int(ids.max()) + 1 if len(ids) else a1)
        # C2 on the re-cut windows: own entries carry their global id; halos must receive theirs
        win = torch.tensor([sh.w0, sh.w1], dtype=torch.int64)
        allw = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allw, win)
        windows = [tuple(int(x) for x in w.tolist()) for w in allw]
        hm = balance.halo_moves(cuts, windows)
        buf = torch.full((sh.w1 - sh.w0, 3), -1.0)
        buf[sh.halo_lo:sh.halo_lo + sh.n_points, 0] = torch.arange(a0, a1, dtype=torch.float32)
        shard_halo_exchange(buf, windows, hm, rank)
        np.testing.assert_array_equal(buf[:, 0].numpy(), np.arange(sh.w0, sh.w1, dtype=np.float32))
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_balanced_repartition(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def test_balanced_layer_cuts():
    """dist.balanced_layer_cuts: contiguous layer ranges covering every layer, >= 1 layer per rank, each
    rank's points within one layer of the ideal share P/world (SURVEY 8(e) point-balanced slabs)."""
    import random
    from paper_2401_14906_b200.dist import balanced_layer_cuts
    rng = random.Random(3)
    cases = [[0] * 10, [5] * 7, [0, 0, 100, 0, 0, 0, 1, 1], [rng.randint(0, 50) for _ in range(200)],
             [int(1000 * (1 - abs(k - 500) / 500)) for k in range(1023)]]
    for pts in cases:
        for world in (1, 2, 3, 4, 8):
            if world > len(pts):
                continue
            cuts = balanced_layer_cuts(pts, world)
            assert cuts[0][0] == 0 and cuts[-1][1] == len(pts)
            assert all(a < b for a, b in cuts) and all(cuts[i][1] == cuts[i + 1][0] for i in range(world - 1))
            tot = sum(pts)
            if tot and world > 1:
                share = tot / world
                for a, b in cuts:
                    assert sum(pts[a:b]) <= share + max(pts) + 1e-9
