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
