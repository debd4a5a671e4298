"""Multi-GPU z-slab decomposition (PSN "can be
run in distributed fashion across multiple sub-volumes" with open boundaries).

One process per GPU.  Rank r owns voxel layers [k0, k1) of the global volume
and holds lattice slices [max(k0-1,0), min(k1+1,O-1)] (a one-slice halo on each
interior side).  The path has two real exchange steps:

  C1  after PSN_COUNT: all-gather of (P_r, Q_r, S_r, halo_lo_r, halo_hi_r) and an
      exclusive scan -> this rank's global first point / quad / stencil ids.
      Because ids are k-major, the rank-order concatenation of every rank's
      output is bit-identical to the single-GPU output.
  C2  after every smoothing iteration: the offsets of the first own voxel layer
      go to rank r-1 (its upper halo), those of the last own layer to rank r+1
      (its lower halo).  The exchange after the last iteration is the final
      halo refresh (C3) needed by triangulation.

  C4  (balance=True) once per step after extraction: the point-balanced
      re-partition of the smoothing work (balance.py): equal global-id shares,
      the moved points' face masks / CSR rows / anchors sent point-to-point to
      their new owners; C2 then runs on the re-cut windows.

The collectives use torch.distributed (NCCL on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import balance


def partition(n_layers: int, world: int):
    """Equal contiguous split of voxel layers [0, n_layers) into `world` ranges."""
    return [(r * n_layers // world, (r + 1) * n_layers // world) for r in range(world)]


def slab_slices(O: int, k0: int, k1: int):
    """Lattice slices [z_lo, z_hi) a rank owning voxel layers [k0, k1) must hold."""
    return max(k0 - 1, 0), min(k1 + 1, O - 1) + 1


def exchange_totals(P: int, Q: int, S: int, halo_lo: int, halo_hi: int, device, group=None):
    """C1: all-gather the per-rank totals; return (first_point, first_quad,
    first_stencil, table) where table[r] = (P, Q, S, halo_lo, halo_hi)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = torch.tensor([P, Q, S, halo_lo, halo_hi], dtype=torch.int64, device=device)
    allt = torch.empty(world * 5, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(allt, mine, group=group)
    table = allt.view(world, 5).cpu()
    first = table[:rank, :3].sum(0)
    totals = table[:, :3].sum(0)
    if int(totals.max()) >= 1 << 32:
        raise OverflowError(f"global totals exceed 32-bit ids: {totals.tolist()}")
    return int(first[0]), int(first[1]), int(first[2]), table


def halo_plan(table, rank: int):
    """Window index ranges exchanged by rank `rank` each smoothing iteration.

    Returns dict with send_lo (own first layer -> rank-1), recv_lo (halo_lo <- rank-1),
    send_hi (own last layer -> rank+1), recv_hi (halo_hi <- rank+1); each (start, stop)
    or None.  The sizes come from the neighbours' halo counts: rank r-1's upper halo is
    exactly rank r's first own layer, and so on.
    """
    world = table.shape[0]
    P, _, _, hl, hh = (int(x) for x in table[rank])
    plan = {"send_lo": None, "recv_lo": None, "send_hi": None, "recv_hi": None}
    if rank > 0:
        n_first = int(table[rank - 1][4])         # rank-1's halo_hi = my first own layer
        plan["send_lo"] = (hl, hl + n_first)
        plan["recv_lo"] = (0, hl)
    if rank < world - 1:
        n_last = int(table[rank + 1][3])          # rank+1's halo_lo = my last own layer
        plan["send_hi"] = (hl + P - n_last, hl + P)
        plan["recv_hi"] = (hl + P, hl + P + hh)
    return plan


def halo_exchange(buf: torch.Tensor, plan, rank: int, group=None):
    """C2/C3: send the boundary layers of `buf` ([n_window, 4] float4 offsets) and receive the halos.
    NCCL point-to-point in one group (batch_isend_irecv)."""
    ops = []
    if plan["send_lo"] is not None:
        a, b = plan["send_lo"]
        c, d = plan["recv_lo"]
        if b > a:
            ops.append(dist.P2POp(dist.isend, buf[a:b], rank - 1, group))
        if d > c:
            ops.append(dist.P2POp(dist.irecv, buf[c:d], rank - 1, group))
    if plan["send_hi"] is not None:
        a, b = plan["send_hi"]
        c, d = plan["recv_hi"]
        if b > a:
            ops.append(dist.P2POp(dist.isend, buf[a:b], rank + 1, group))
        if d > c:
            ops.append(dist.P2POp(dist.irecv, buf[c:d], rank + 1, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


class SlabPipeline:
    """One rank's slab: extraction with halos + smoothing with halo exchange.

    Used by bench.py for N > 1 (and by the 1-GPU slab-emulation tests through
    the same psn_extract / psn_smooth_step calls)."""

    def __init__(self, psn, labels_slab: torch.Tensor, dims, spacing, origin, own, iterations, relaxation,
                 constraint, label_set=None, group=None):
        from .psn import MeshC
        self.psn, self.group = psn, group
        self.rank = dist.get_rank(group)
        z_lo = slab_slices(dims[2], own[0], own[1])[0]
        self.vol = psn.volume(labels_slab, dims=dims, spacing=spacing, origin=origin, z_lo=z_lo, own=own)
        self.labels = psn.labels(label_set)
        self.T, self.lam, self.d = iterations, relaxation, constraint
        self.ws = psn.workspace(self.vol)
        c = psn.count(self.vol, self.labels, self.ws)
        self.first_point, self.first_quad, self.first_stencil, self.table = exchange_totals(
            c.n_points, c.n_quads, c.n_stencil, c.halo_lo_points, c.halo_hi_points, labels_slab.device, group)
        self.mesh = psn.emit(self.vol, self.labels, self.ws, c,
                             first=(self.first_point, self.first_quad, self.first_stencil))
        self.counted = MeshC.from_buffer_copy(self.mesh.c)
        self.plan = halo_plan(self.table, self.rank)
        nw = self.mesh.n_window
        self.sws = psn.smooth_workspace(self.mesh)
        self.buf = [psn.offsets_buffer(nw, labels_slab.device) for _ in range(2)]   # float4 offsets
        self.out = torch.empty((max(nw, 1), 3), dtype=torch.float32, device=labels_slab.device)

    def extract(self, stream=None):
        """Per-step extraction: COUNT -> C1 (all-gather) -> EMIT (one host sync for the totals)."""
        c = self.psn.count(self.vol, self.labels, self.ws, stream)
        self.first_point, self.first_quad, self.first_stencil, self.table = exchange_totals(
            c.n_points, c.n_quads, c.n_stencil, c.halo_lo_points, c.halo_hi_points, self.buf[0].device, self.group)
        self.psn.emit(self.vol, self.labels, self.ws, c, first=(self.first_point, self.first_quad, self.first_stencil),
                      mesh=self.mesh, stream=stream)

    def smooth_balanced(self, stream=None):
        """C4 (point-balanced re-partition of this step's mesh) + T Jacobi steps on the
        re-cut shards with their halo exchange; returns this rank's share of the
        global smoothed points (ids [cuts[rank], cuts[rank+1]))."""
        total = int(self.table[:, 0].sum())
        self.balanced = BalancedSmoother(self.psn, self.vol, self.mesh, self.first_point, self.first_stencil, total,
                                         self.T, self.lam, self.d, self.group)
        return self.balanced.smooth(stream)

    def smooth(self, stream=None):
        """T Jacobi steps with a halo exchange after each (C2; the last one is C3)."""
        src = None
        self.psn.smooth_prepare(self.vol, self.mesh, self.sws, stream)
        for t in range(self.T):
            dst = self.buf[t & 1]
            self.psn.smooth_step(self.vol, self.mesh, self.sws, src, dst, self.lam, self.d, stream)
            halo_exchange(dst, self.plan, self.rank, self.group)
            src = dst
        self.psn.smooth_finalize(self.vol, self.mesh, src, self.out, 0, self.mesh.n_window, stream)
        return self.out


def p2p_transport(group=None):
    """balance.assemble transport over torch.distributed point-to-point (blocking
    send / recv in the common move order: every move involves exactly its two
    ranks, so the sequence cannot deadlock)."""
    me = dist.get_rank(group)

    def transport(src, dst, tensor, like):
        if src == dst:
            return tensor if me == src else None
        if me == src:
            dist.send(tensor, dst, group=group)
            return None
        if me == dst:
            dist.recv(like, src, group=group)
            return like
        return None
    return transport


def shard_halo_exchange(buf: torch.Tensor, shard_windows, moves, rank: int, group=None):
    """C2 on re-cut windows: for every halo move (src, dst, g0, g1), src sends its
    window slice of ids [g0, g1) to dst's window slice (batched P2P)."""
    ops = []
    for (s, d, g0, g1) in moves:
        if s == rank:
            w0 = shard_windows[s][0]
            ops.append(dist.P2POp(dist.isend, buf[g0 - w0:g1 - w0], d, group))
        elif d == rank:
            w0 = shard_windows[d][0]
            ops.append(dist.P2POp(dist.irecv, buf[g0 - w0:g1 - w0], s, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


class BalancedSmoother:
    """C4 + smoothing on the point-balanced shards: built from a
    rank's extraction (SlabPipeline) after C1; smooth() runs T psn_smooth_step
    iterations with the halo exchange of the re-cut windows and returns the
    world coordinates of this rank's own ids [cuts[rank], cuts[rank+1])."""

    def __init__(self, psn, vol, mesh, first_point: int, first_stencil: int, total_points: int, iterations: int,
                 relaxation: float, constraint: float, group=None):
        self.psn, self.vol, self.group = psn, vol, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.T, self.lam, self.d = iterations, relaxation, constraint
        dev = mesh.points.device
        src = balance.source_from_mesh(mesh, first_point, first_stencil)
        owned = torch.tensor([first_point, mesh.n_points], dtype=torch.int64, device=dev)
        allo = torch.empty(2 * self.world, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(allo, owned, group=group)
        owned_all = [tuple(int(x) for x in allo[2 * r:2 * r + 2].tolist()) for r in range(self.world)]
        self.cuts = balance.balanced_cuts(total_points, self.world)
        moves = balance.plan_moves(owned_all, self.cuts)
        self.shard = balance.assemble(self.rank, self.cuts, moves, src, p2p_transport(group), dev)
        win = torch.tensor([self.shard.w0, self.shard.w1], dtype=torch.int64, device=dev)
        allw = torch.empty(2 * self.world, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(allw, win, group=group)
        self.windows = [tuple(int(x) for x in allw[2 * r:2 * r + 2].tolist()) for r in range(self.world)]
        self.halo = balance.halo_moves(self.cuts, self.windows)
        self.mesh = balance.shard_mesh(psn, self.shard)
        nw = max(self.shard.w1 - self.shard.w0, 1)
        self.sws = psn.smooth_workspace(self.mesh)
        self.buf = [psn.offsets_buffer(nw, dev) for _ in range(2)]   # float4 offsets
        self.out = torch.empty((nw, 3), dtype=torch.float32, device=dev)

    def smooth(self, stream=None):
        sh = self.shard
        src = None
        if sh.n_points:
            self.psn.smooth_prepare(self.vol, self.mesh, self.sws, stream)
        for t in range(self.T):
            dst = self.buf[t & 1]
            if sh.n_points:
                self.psn.smooth_step(self.vol, self.mesh, self.sws, src, dst, self.lam, self.d, stream)
            shard_halo_exchange(dst, self.windows, self.halo, self.rank, self.group)
            src = dst
        if sh.n_points:
            self.psn.smooth_finalize(self.vol, self.mesh, src, self.out, sh.halo_lo, sh.halo_lo + sh.n_points, stream)
        return self.out[sh.halo_lo:sh.halo_lo + sh.n_points]
