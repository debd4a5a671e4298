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

  C2 v2 (peer=True, SV 8(e) v2): the halo exchange is fused into the smoothing
      kernel -- psn_smooth_step_peer stores the boundary layers it computes
      straight into the neighbours' offset buffers over NVLink (CUDA IPC peer
      pointers, exchanged once) and signals them; a step starts once both
      neighbours finished the previous one.  No collective and no host sync
      in the iteration loop.  Used when every halo move is between adjacent
      ranks (always for slabs; for balanced shards in practice), else C2 over
      NCCL.

The collectives use torch.distributed (NCCL on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import balance


def partition(n_layers: int, world: int):
    """Equal contiguous split of voxel layers [0, n_layers) into `world` ranges."""
    return [(r * n_layers // world, (r + 1) * n_layers // world) for r in range(world)]


def balanced_layer_cuts(layer_points, world: int):
    """Contiguous voxel-layer ranges with (nearly) equal point counts: rank r owns
    layers [c_r, c_{r+1}) where c_r is the first layer whose exclusive point prefix reaches
    r * P / world; every rank owns >= 1 layer.  `layer_points` = points per voxel layer of the
    whole volume (the same list on every rank, so the cuts agree without a collective)."""
    n = len(layer_points)
    if world > n:
        raise ValueError("more ranks than voxel layers")
    total = sum(int(x) for x in layer_points)
    cuts, acc, r = [0], 0, 1
    for k, x in enumerate(layer_points):
        # cut before layer k when the points so far reach rank r's share (and layers remain for the rest)
        while r < world and acc * world >= r * total and k > cuts[-1] and n - k >= world - r:
            cuts.append(k)
            r += 1
        acc += int(x)
    while r < world:   # degenerate (e.g. no points): equal layers for the remaining ranks
        cuts.append(max(cuts[-1] + 1, (r * n) // world))
        r += 1
    cuts.append(n)
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


def gather_layer_points(psn, vol, ws, own, group=None):
    """All-gather every rank's per-layer point counts of its own layers (C1 widened, SURVEY 8(e):
    ~4 B per layer) -> the whole volume's per-layer list (rank order = layer order)."""
    counts, _ = psn.rows(vol, ws)
    N = vol.dims[1]
    kA = own[0] - (1 if own[0] > 0 else 0)
    P = counts[0].to(torch.int64).view(-1, N - 1).sum(1)[own[0] - kA: own[1] - kA]
    world = dist.get_world_size(group)
    n = torch.tensor([P.numel()], dtype=torch.int64, device=P.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    m = int(max(int(x.item()) for x in ns))
    pad = torch.zeros(m, dtype=torch.int64, device=P.device)
    pad[:P.numel()] = P
    outs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    res = []
    for o, k in zip(outs, ns):
        res += o[:int(k.item())].tolist()
    return res


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


def peer_sides(rank: int, world: int, sends):
    """Symmetric peer-push plan for psn_smooth_step_peer.

    sends: [(src, dst, src_begin, src_end, dst_begin)] -- every rank's pushes,
    window index ranges in src's window and the receiving index in dst's window
    (the same list on all ranks).  Returns (lower, upper) for `rank`: None if
    there is no exchange with that neighbour, else (src_begin, src_end,
    dst_begin) of this rank's push to it (an empty range when only the
    neighbour pushes here -- the signal still has to flow both ways, because a
    rank may only push into a neighbour that has finished the previous step).
    Raises ValueError if a push is not between adjacent ranks or a rank pushes
    two ranges to one neighbour (the caller then falls back to NCCL)."""
    out = {}
    touch = set()
    for (sr, dr, a, b, c) in sends:
        if b <= a:
            continue
        if abs(sr - dr) != 1:
            raise ValueError(f"push {sr}->{dr} is not between adjacent ranks")
        if (sr, dr) in out:
            raise ValueError(f"rank {sr} pushes two ranges to {dr}")
        out[(sr, dr)] = (a, b, c)
        touch.add((min(sr, dr), max(sr, dr)))
    res = []
    for nb in (rank - 1, rank + 1):
        if nb < 0 or nb >= world or (min(rank, nb), max(rank, nb)) not in touch:
            res.append(None)
            continue
        res.append(out.get((rank, nb), (0, 0, 0)))
    return res[0], res[1]


def slab_sends(table):
    """Peer pushes of the z-slab halo plan: rank r's first own layer -> rank r-1's
    upper halo, its last own layer -> rank r+1's lower halo."""
    world = table.shape[0]
    sends = []
    for r in range(world):
        pl = halo_plan(table, r)
        if pl["send_lo"] is not None:
            a, b = pl["send_lo"]
            c, _ = halo_plan(table, r - 1)["recv_hi"]
            sends.append((r, r - 1, a, b, c))
        if pl["send_hi"] is not None:
            a, b = pl["send_hi"]
            c, _ = halo_plan(table, r + 1)["recv_lo"]
            sends.append((r, r + 1, a, b, c))
    return sends


def shard_sends(halo, windows):
    """Peer pushes of the balanced shards: halo move (src, dst, g0, g1) of global ids
    -> (src, dst, g0 - w0[src], g1 - w0[src], g0 - w0[dst])."""
    return [(s_, d_, g0 - windows[s_][0], g1 - windows[s_][0], g0 - windows[d_][0]) for (s_, d_, g0, g1) in halo]


class PeerHalo:
    """The peer-push state of one rank (psn_smooth_step_peer): its two float4
    offset buffers and signal words exported once over CUDA IPC, the
    neighbours' mapped, and the psn_peer descriptor advanced by every step."""

    def __init__(self, psn, bufs, lower, upper, group=None):
        from .psn import Peer
        self.psn, self.bufs = psn, bufs
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        dev = bufs[0].device
        self.sig = torch.zeros(2, dtype=torch.int64, device=dev)     # u64 words, written by the neighbours
        self.ctr = torch.zeros(1, dtype=torch.int64, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        torch.cuda.synchronize(dev)   # zeroed before any neighbour can signal
        try:
            mine = [psn.ipc_export(bufs[0]), psn.ipc_export(bufs[1]), psn.ipc_export(self.sig)]
        except Exception:   # e.g. memory not from cudaMalloc: every rank must then fall back together
            mine = None
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        if any(h is None for h in allh):
            raise ValueError("CUDA IPC export failed on some rank")
        self.peer = Peer()
        self.peer.sig, self.peer.ctr, self.peer.err = self.sig.data_ptr(), self.ctr.data_ptr(), self.err.data_ptr()
        self.opened = []
        ok = True
        try:
            for k, (nb, spec) in enumerate(((rank - 1, lower), (rank + 1, upper))):
                if spec is None:
                    continue
                b0, b1, sg = (psn.ipc_open(h) for h in allh[nb])
                self.opened += [b0, b1, sg]
                side = self.peer.side[k]
                side.dst[0], side.dst[1] = b0, b1
                side.src_begin, side.src_end, side.dst_begin = spec
                side.peer_sig = sg + 8 * (1 - k)   # pushes down land in the lower rank's sig[1], up in sig[0]
        except Exception:
            ok = False
        oks = [None] * world
        dist.all_gather_object(oks, ok, group=group)   # also: every rank mapped its neighbours before anyone signals
        if not all(oks):
            self.close()
            raise ValueError("CUDA IPC open failed on some rank")

    def step(self, vol, mesh, ws, src, dst, parity, lam, d, stream=None):
        self.psn.smooth_step_peer(vol, mesh, ws, src, dst, parity, lam, d, self.peer, stream)

    def run(self, vol, mesh, ws, iterations, lam, d, stream=None):
        """All iterations in one library call (one launch each, no host round trip per step)."""
        return self.psn.smooth_run_peer(vol, mesh, ws, self.bufs, iterations, lam, d, self.peer, stream)

    def check(self):
        if int(self.err.item()):
            raise RuntimeError("peer halo wait timed out (a neighbour stopped stepping)")

    def close(self):
        for a in self.opened:
            self.psn.ipc_close(a)
        self.opened = []


class SlabPipeline:
    """One rank's slab: extraction with halos + smoothing with halo exchange.

    Used by bench.py for N > 1 (and by the 1-GPU slab-emulation tests through
    the same psn_extract / psn_smooth_step calls)."""

    def __init__(self, psn, labels_slab: torch.Tensor, dims, spacing, origin, own, iterations, relaxation,
                 constraint, label_set=None, group=None, peer: bool = False):
        from .psn import MeshC
        self.psn, self.group, self.use_peer = psn, group, peer
        self.peer_halo, self._shard_cache = None, {}
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
        # device-side C1 for the steady-state steps (NCCL): COUNT|DEVICE -> totals -> all-gather ->
        # prefix sum -> EMIT|DEVICE, no host round trip; the mesh's host fields stay those of this count
        self.device_c1 = dist.get_backend(group) == "nccl"
        dev = labels_slab.device
        self._tot = torch.zeros(5, dtype=torch.int64, device=dev)
        self._all = torch.zeros(5 * dist.get_world_size(group), dtype=torch.int64, device=dev)
        self._first = torch.zeros(3, dtype=torch.int64, device=dev)
        nw = self.mesh.n_window
        self.sws = psn.smooth_workspace(self.mesh)
        self.buf = [psn.offsets_buffer(nw, labels_slab.device) for _ in range(2)]   # float4 offsets
        self.out = torch.empty((max(nw, 1), 3), dtype=torch.float32, device=labels_slab.device)

    def extract(self, stream=None):
        """Per-step extraction: COUNT -> C1 (all-gather) -> EMIT.  With NCCL all three stay on the
        device (steady state: the volume's totals are those of the setup count, checked by
        check_totals()); otherwise one host sync reads the totals."""
        if self.device_c1:
            world = dist.get_world_size(self.group)
            self.psn.count_device(self.vol, self.labels, self.ws, self._tot, stream)
            dist.all_gather_into_tensor(self._all, self._tot, group=self.group)
            torch.sum(self._all.view(world, 5)[:self.rank, :3], 0, out=self._first)
            self.psn.emit_device(self.vol, self.labels, self.ws, self.mesh, self._first, stream)
            return
        c = self.psn.count(self.vol, self.labels, self.ws, stream)
        self.first_point, self.first_quad, self.first_stencil, self.table = exchange_totals(
            c.n_points, c.n_quads, c.n_stencil, c.halo_lo_points, c.halo_hi_points, self.buf[0].device, self.group)
        self.psn.emit(self.vol, self.labels, self.ws, c, first=(self.first_point, self.first_quad, self.first_stencil),
                      mesh=self.mesh, stream=stream)

    def check_totals(self):
        """Synchronising check that the device-side C1 of the last step saw the setup's per-rank totals
        (the mesh's host fields and the halo plan assume them) and no emission was skipped."""
        if self.device_c1:
            got = self._all.view(-1, 5).cpu()
            if not torch.equal(got, self.table.to(got.dtype)):
                raise RuntimeError("per-rank totals changed since the setup count: rebuild the SlabPipeline")
        self.psn.totals(self.vol, self.ws, self.mesh)

    def smooth_balanced(self, stream=None):
        """C4 (point-balanced re-partition of this step's mesh) + T Jacobi steps on the
        re-cut shards with their halo exchange; returns this rank's share of the
        global smoothed points (ids [cuts[rank], cuts[rank+1]))."""
        total = int(self.table[:, 0].sum())
        # the ranks' owned id ranges follow from C1's table (no extra all-gather)
        P = [int(x) for x in self.table[:, 0].tolist()]
        owned = [(sum(P[:r]), P[r]) for r in range(len(P))]
        self.balanced = BalancedSmoother(self.psn, self.vol, self.mesh, self.first_point, self.first_stencil, total,
                                         self.T, self.lam, self.d, self.group, peer=self.use_peer,
                                         cache=self._shard_cache, owned_all=owned)
        return self.balanced.smooth(stream)

    def smooth(self, stream=None):
        """T Jacobi steps with a halo exchange after each (C2; the last one is C3):
        fused into the step kernel (peer pushes) when peer=True, else NCCL."""
        src = None
        self.psn.smooth_prepare(self.vol, self.mesh, self.sws, stream)
        if self.use_peer:
            key = self.table.numpy().tobytes()   # halo sizes follow this step's per-rank counts
            if self.peer_halo is None or self._peer_key != key:
                if self.peer_halo is not None:
                    self.peer_halo.close()
                try:
                    lower, upper = peer_sides(self.rank, dist.get_world_size(self.group), slab_sends(self.table))
                    self.peer_halo, self._peer_key = PeerHalo(self.psn, self.buf, lower, upper, self.group), key
                except ValueError:   # consistent on every rank: C2 over NCCL from now on
                    self.use_peer, self.peer_halo = False, None
        if self.use_peer and self.peer_halo is not None:
            src = self.peer_halo.run(self.vol, self.mesh, self.sws, self.T, self.lam, self.d, stream)
        for t in range(0 if self.use_peer else self.T):
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


def assemble_batched(rank: int, cuts, moves, source, device, group=None):
    """balance.assemble with the point-to-point traffic in two batches instead of one
    blocking send / recv per array: (1) every move's stencil-id count, (2) every
    move's five arrays.  All ranks walk `moves` in the same order, so the posted
    sends and receives of each rank pair match.  Zero-length arrays are skipped
    on both sides (their sizes are known to both after batch 1)."""
    mine = [(k, mv) for k, mv in enumerate(moves) if rank in (mv[0], mv[1])]
    pieces, cnts, ops = {}, {}, []
    for k, (s_, d_, g0, g1) in mine:
        if s_ == rank:
            pieces[k] = source.piece(g0, g1)
            cnts[k] = torch.tensor([pieces[k]["stencil_ids"].numel()], dtype=torch.int64, device=device)
            if d_ != rank:
                ops.append(dist.P2POp(dist.isend, cnts[k], d_, group))
        else:
            cnts[k] = torch.empty(1, dtype=torch.int64, device=device)
            ops.append(dist.P2POp(dist.irecv, cnts[k], s_, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    ops, parts = [], []
    keys = ("face_masks", "stencil_offsets", "stencil_ids", "points", "end_offset")
    for k, (s_, d_, g0, g1) in mine:
        if s_ == rank and d_ == rank:
            parts.append((g0, g1, pieces[k]))
            continue
        n, c = g1 - g0, int(cnts[k].item())
        if s_ == rank:
            for key in keys:
                t = pieces[k][key].contiguous()
                if t.numel():
                    ops.append(dist.P2POp(dist.isend, t, d_, group))
        else:
            like = dict(face_masks=torch.empty(n, dtype=torch.uint8, device=device),
                        stencil_offsets=torch.empty(n, dtype=torch.int32, device=device),
                        stencil_ids=torch.empty(c, dtype=torch.int32, device=device),
                        points=torch.empty((n, 3), dtype=torch.float32, device=device),
                        end_offset=torch.empty(1, dtype=torch.int32, device=device))
            for key in keys:
                if like[key].numel():
                    ops.append(dist.P2POp(dist.irecv, like[key], s_, group))
            parts.append((g0, g1, like))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return balance._finish(balance.Shard(cuts[rank], cuts[rank + 1]), parts, device)


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
                 relaxation: float, constraint: float, group=None, peer: bool = False, cache=None, owned_all=None):
        self.psn, self.vol, self.group = psn, vol, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.T, self.lam, self.d = iterations, relaxation, constraint
        dev = mesh.points.device
        src = balance.source_from_mesh(mesh, first_point, first_stencil)
        if owned_all is None:   # (callers with C1's table pass it: no collective here)
            owned = torch.tensor([first_point, mesh.n_points], dtype=torch.int64, device=dev)
            allo = torch.empty(2 * self.world, dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(allo, owned, group=group)
            owned_all = [tuple(int(x) for x in allo[2 * r:2 * r + 2].tolist()) for r in range(self.world)]
        self.cuts = balance.balanced_cuts(total_points, self.world)
        moves = balance.plan_moves(owned_all, self.cuts)
        self.shard = assemble_batched(self.rank, self.cuts, moves, src, dev, group)
        win = torch.tensor([self.shard.w0, self.shard.w1], dtype=torch.int64, device=dev)
        allw = torch.empty(2 * self.world, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(allw, win, group=group)
        self.windows = [tuple(int(x) for x in allw[2 * r:2 * r + 2].tolist()) for r in range(self.world)]
        self.halo = balance.halo_moves(self.cuts, self.windows)
        self.mesh = balance.shard_mesh(psn, self.shard)
        nw = max(self.shard.w1 - self.shard.w0, 1)
        self.peer = None
        key = (tuple(self.cuts), tuple(self.windows))
        if cache is not None and key in cache:   # same shard layout as an earlier step: reuse buffers, IPC maps,
            self.buf, self.peer, self.sws, self.out = cache[key]   # workspace and output
        else:
            self.sws = psn.smooth_workspace(self.mesh)
            self.out = torch.empty((nw, 3), dtype=torch.float32, device=dev)
            self.buf = [psn.offsets_buffer(nw, dev) for _ in range(2)]   # float4 offsets
            if peer:
                try:
                    lower, upper = peer_sides(self.rank, self.world, shard_sends(self.halo, self.windows))
                    self.peer = PeerHalo(psn, self.buf, lower, upper, group)
                except ValueError:
                    self.peer = None   # a non-adjacent halo move: C2 over NCCL
            if cache is not None:
                for ent in cache.values():
                    if ent[1] is not None:
                        ent[1].close()
                cache.clear()
                cache[key] = (self.buf, self.peer, self.sws, self.out)

    def smooth(self, stream=None):
        sh = self.shard
        src = None
        if sh.n_points:
            self.psn.smooth_prepare(self.vol, self.mesh, self.sws, stream)
        if self.peer is not None:   # the steps' kernels push the halos (every rank steps, even empty ones)
            src = self.peer.run(self.vol, self.mesh, self.sws, self.T, self.lam, self.d, stream)
        for t in range(0 if self.peer is not None else self.T):
            dst = self.buf[t & 1]
            if sh.n_points:
                self.psn.smooth_step(self.vol, self.mesh, self.sws, src, dst, self.lam, self.d, stream)
            shard_halo_exchange(dst, self.windows, self.halo, self.rank, self.group)
            src = dst
        if sh.n_points:
            self.psn.smooth_finalize(self.vol, self.mesh, src, self.out, sh.halo_lo, sh.halo_lo + sh.n_points, stream)
        return self.out[sh.halo_lo:sh.halo_lo + sh.n_points]
