"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): partition, C1
(all-gather + exclusive scan of per-rank totals) and C2 (halo exchange plan and
point-to-point exchange).  The GPU kernels are exercised by
tests/test_gpu_slabs.py; here the buffers are CPU tensors and each rank fills
its own entries with recognisable values."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_14906_b200.dist import exchange_totals, halo_exchange, halo_plan, partition, slab_slices


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, layer_points, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O = len(layer_points) + 1
        k0, k1 = partition(O - 1, world)[rank]
        P = sum(layer_points[k0:k1])
        hl = layer_points[k0 - 1] if k0 > 0 else 0
        hh = layer_points[k1] if k1 < O - 1 else 0
        fp, fq, fs, table = exchange_totals(P, 2 * P, 4 * P, hl, hh, torch.device("cpu"))
        assert fp == sum(layer_points[:k0])
        assert (fq, fs) == (2 * fp, 4 * fp)
        plan = halo_plan(table, rank)
        nw = hl + P + hh
        buf = torch.full((nw, 3), -1.0)
        # own entries: the global id of the point
        gid0 = fp
        buf[hl:hl + P, 0] = torch.arange(gid0, gid0 + P, dtype=torch.float32)
        halo_exchange(buf, plan, rank)
        # halos now hold the neighbours' global ids: layer k0-1 ends at fp-1, layer k1 starts at fp+P
        if hl:
            assert torch.equal(buf[:hl, 0], torch.arange(fp - hl, fp, dtype=torch.float32))
        if hh:
            assert torch.equal(buf[hl + P:, 0], torch.arange(fp + P, fp + P + hh, dtype=torch.float32))
        z_lo, z_hi = slab_slices(O, k0, k1)
        assert z_lo == max(k0 - 1, 0) and z_hi == min(k1 + 1, O - 1) + 1
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_totals_and_halo_exchange(world):
    layer_points = [3, 0, 5, 7, 2, 9, 4, 6, 1, 8]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layer_points, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def test_partition_covers_layers():
    for n, w in [(1023, 8), (7, 3), (5, 5)]:
        parts = partition(n, w)
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


# ---------------------------------------------------------------- peer-push planning (SV 8(e) v2)
def test_peer_sides_slabs_match_halo_plan():
    """slab_sends / peer_sides give every rank exactly its halo_plan send ranges,
    landing at the neighbour's receive ranges, and both neighbours see each other."""
    from paper_2401_14906_b200.dist import halo_plan, peer_sides, slab_sends
    table = torch.tensor([[100, 0, 0, 0, 7], [120, 0, 0, 9, 11], [90, 0, 0, 13, 5], [80, 0, 0, 6, 0]])
    G = table.shape[0]
    sends = slab_sends(table)
    for r in range(G):
        lower, upper = peer_sides(r, G, sends)
        pl = halo_plan(table, r)
        if r == 0:
            assert lower is None
        else:
            a, b = pl["send_lo"]
            c, d = halo_plan(table, r - 1)["recv_hi"]
            assert lower == (a, b, c) and d - c == b - a
        if r == G - 1:
            assert upper is None
        else:
            a, b = pl["send_hi"]
            c, d = halo_plan(table, r + 1)["recv_lo"]
            assert upper == (a, b, c) and d - c == b - a


def test_peer_sides_symmetric_and_rejects_non_adjacent():
    from paper_2401_14906_b200.dist import peer_sides
    # only rank 1 pushes to rank 2: rank 2 still gets a side (empty range) so signals flow both ways
    sends = [(1, 2, 10, 20, 0)]
    assert peer_sides(1, 3, sends) == (None, (10, 20, 0))
    assert peer_sides(2, 3, sends) == ((0, 0, 0), None)
    assert peer_sides(0, 3, sends) == (None, None)
    with pytest.raises(ValueError):
        peer_sides(0, 3, [(0, 2, 0, 5, 0)])
    with pytest.raises(ValueError):
        peer_sides(0, 3, [(0, 1, 0, 5, 0), (0, 1, 7, 9, 3)])


def test_peer_sides_balanced_shards():
    """shard_sends of balanced cuts: pushes are own ids of the sender, land inside the
    receiver's halo, and are between adjacent ranks."""
    from paper_2401_14906_b200 import balance
    from paper_2401_14906_b200.dist import peer_sides, shard_sends
    cuts = balance.balanced_cuts(1000, 4)
    windows = [(max(0, cuts[r] - 40), min(1000, cuts[r + 1] + 40)) for r in range(4)]
    hm = balance.halo_moves(cuts, windows)
    sends = shard_sends(hm, windows)
    for (s_, d_, a, b, c) in sends:
        assert abs(s_ - d_) == 1
        g0 = a + windows[s_][0]
        assert cuts[s_] <= g0 and b + windows[s_][0] <= cuts[s_ + 1]
        assert windows[d_][0] + c == g0
        dst_own = (cuts[d_] - windows[d_][0], cuts[d_ + 1] - windows[d_][0])
        assert c + (b - a) <= dst_own[0] or c >= dst_own[1]   # into the halo, not the own range
    for r in range(4):
        lower, upper = peer_sides(r, 4, sends)
        assert (lower is None) == (r == 0) and (upper is None) == (r == 3)
