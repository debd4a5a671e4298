"""Point-balanced re-partition of the smoothing work across ranks.

Extraction partitions the volume into equal z-slabs (balanced label reads), but
surface points are not spread evenly over z: with equal slabs c4's per-rank
point counts reach 1.5x the mean at 8 ranks, which caps smoothing scaling
(Eq. 1's cost is per point).  Because point ids are k-major (reading
Q4), a contiguous id range is a z-slab with partial end layers, so after
extraction every rank can own an equal share of ids for smoothing:

    smoothing owner of ids [A_r, A_{r+1}),  A_r = floor(r * P / G)

Moving a point means moving what psn_smooth_step needs for it: its face mask,
its CSR row (global ids, so no renumbering) and its fp32 anchor (for the final
world coordinates).  Each rank's smoothing window is its own range extended
to the smallest / largest stencil id it references; the per-iteration halo
exchange sends, from every owner, the slices of its own range that fall in
other ranks' windows.  Stencils only reach about one voxel layer away, so with
balanced cuts every exchange is between neighbouring ranks, but the planning
below is general.

Everything here is host-side planning plus tensor slicing; the data moves
through a `transport(src, dst, tensor)` callable (NCCL point-to-point in
dist.py, plain device copies in the one-GPU emulation tests).  No arithmetic of
the method happens here.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


def balanced_cuts(total: int, world: int):
    """A_0 = 0 <= A_1 <= ... <= A_G = total, ranges of (almost) equal size."""
    return [r * total // world for r in range(world + 1)]


def overlap(a0: int, a1: int, b0: int, b1: int):
    lo, hi = max(a0, b0), min(a1, b1)
    return (lo, hi) if hi > lo else None


@dataclass
class SourceMesh:
    """One rank's extraction output (window-indexed as psn_mesh): own global ids
    [first_point, first_point + n_points); points[w] = anchor of id
    first_point - halo_lo + w."""
    first_point: int
    n_points: int
    halo_lo: int
    first_stencil: int
    points: torch.Tensor          # float32 [W, 3]
    face_masks: torch.Tensor      # uint8 [P]
    stencil_offsets: torch.Tensor  # int32 view of uint32 [P + 1] (global)
    stencil_ids: torch.Tensor     # int32 view of uint32 [S] (global ids)

    def piece(self, g0: int, g1: int):
        """The arrays of global ids [g0, g1) (inside this rank's own range)."""
        a, b = g0 - self.first_point, g1 - self.first_point
        off = self.stencil_offsets[a:b + 1]
        s0 = (int(off[0].item()) & 0xFFFFFFFF) - self.first_stencil     # uint32 values in an int32 view
        s1 = (int(off[-1].item()) & 0xFFFFFFFF) - self.first_stencil
        return dict(face_masks=self.face_masks[a:b], stencil_offsets=off[:-1], stencil_ids=self.stencil_ids[s0:s1],
                    points=self.points[self.halo_lo + a:self.halo_lo + b], end_offset=off[-1:])


@dataclass
class Shard:
    """A rank's smoothing shard: own ids [a0, a1) and window [w0, w1) (all ids
    its stencils reference).  Arrays are laid out as a psn_mesh with
    first_point = a0, halo_lo = a0 - w0, halo_hi = w1 - a1."""
    a0: int
    a1: int
    w0: int = 0
    w1: int = 0
    face_masks: torch.Tensor | None = None
    stencil_offsets: torch.Tensor | None = None   # [P + 1], global values
    stencil_ids: torch.Tensor | None = None
    points: torch.Tensor | None = None            # [W, 3]: anchors of the own ids, zeros in the halos

    @property
    def n_points(self):
        return self.a1 - self.a0

    @property
    def halo_lo(self):
        return self.a0 - self.w0

    @property
    def halo_hi(self):
        return self.w1 - self.a1


def plan_moves(owned, cuts):
    """owned[r] = (first_point, n_points) of rank r's extraction; returns
    [(src, dst, g0, g1)] so that every id of [cuts[dst], cuts[dst+1]) comes
    from its extraction owner, in global order per dst."""
    G = len(owned)
    out = []
    for dst in range(G):
        for src in range(G):
            f, p = owned[src]
            o = overlap(f, f + p, cuts[dst], cuts[dst + 1])
            if o:
                out.append((src, dst, o[0], o[1]))
    return out


def _finish(sh: Shard, parts, device) -> Shard:
    """Concatenate the received pieces (global order) into the shard's arrays and window."""
    if sh.n_points == 0:
        sh.w0, sh.w1 = sh.a0, sh.a1
        sh.face_masks = torch.empty(0, dtype=torch.uint8, device=device)
        sh.stencil_offsets = torch.zeros(1, dtype=torch.int32, device=device)
        sh.stencil_ids = torch.empty(0, dtype=torch.int32, device=device)
        sh.points = torch.zeros((0, 3), dtype=torch.float32, device=device)
        return sh
    parts = sorted(parts, key=lambda x: x[0])
    sh.face_masks = torch.cat([p[2]["face_masks"] for p in parts])
    sh.stencil_offsets = torch.cat([p[2]["stencil_offsets"] for p in parts] + [parts[-1][2]["end_offset"]])
    sh.stencil_ids = torch.cat([p[2]["stencil_ids"] for p in parts])
    own_pts = torch.cat([p[2]["points"] for p in parts])
    ids = sh.stencil_ids.to(torch.int64) & 0xFFFFFFFF
    lo = int(ids.min().item()) if ids.numel() else sh.a0
    hi = int(ids.max().item()) + 1 if ids.numel() else sh.a1
    sh.w0, sh.w1 = min(sh.a0, lo), max(sh.a1, hi)
    sh.points = torch.zeros((sh.w1 - sh.w0, 3), dtype=torch.float32, device=device)
    sh.points[sh.halo_lo:sh.halo_lo + sh.n_points] = own_pts
    return sh


def assemble_local(rank: int, cuts, moves, sources, device) -> Shard:
    """One-process version (all ranks' SourceMesh objects at hand): the shard of `rank`."""
    parts = [(g0, g1, sources[src].piece(g0, g1)) for (src, dst, g0, g1) in moves if dst == rank]
    return _finish(Shard(cuts[rank], cuts[rank + 1]), parts, device)


def assemble(rank: int, cuts, moves, source: SourceMesh, transport, device) -> Shard:
    """Distributed version: every rank calls this with the same `moves`; for each
    move the source rank ships the piece's arrays through
    `transport(src, dst, tensor_or_None, recv_buffer)`, which returns the tensor
    on dst (and on a src == dst move), None elsewhere."""
    parts = []
    for (src, dst, g0, g1) in moves:
        if rank != src and rank != dst:
            continue
        n = g1 - g0
        mine = source.piece(g0, g1) if src == rank else None
        # the receiver learns the piece's stencil-id count first
        cnt = torch.tensor([mine["stencil_ids"].numel() if mine is not None else 0], dtype=torch.int64, device=device)
        cnt = transport(src, dst, cnt if mine is not None else None, cnt)
        like = dict(face_masks=torch.empty(n, dtype=torch.uint8, device=device),
                    stencil_offsets=torch.empty(n, dtype=torch.int32, device=device),
                    stencil_ids=torch.empty(int(cnt.item()) if cnt is not None else 0, dtype=torch.int32, device=device),
                    points=torch.empty((n, 3), dtype=torch.float32, device=device),
                    end_offset=torch.empty(1, dtype=torch.int32, device=device))
        recv = {}
        for k in ("face_masks", "stencil_offsets", "stencil_ids", "points", "end_offset"):
            t = transport(src, dst, None if mine is None else mine[k].contiguous(), like[k])
            if dst == rank:
                recv[k] = t
        if dst == rank:
            parts.append((g0, g1, recv))
    return _finish(Shard(cuts[rank], cuts[rank + 1]), parts, device)


def halo_moves(cuts, windows):
    """windows[r] = (w0, w1).  Returns [(src, dst, g0, g1)]: ids owned by src
    that lie in dst's halo (its window minus its own range)."""
    G = len(windows)
    out = []
    for dst in range(G):
        w0, w1 = windows[dst]
        for (h0, h1) in ((w0, cuts[dst]), (cuts[dst + 1], w1)):
            if h1 <= h0:
                continue
            for src in range(G):
                if src == dst:
                    continue
                o = overlap(h0, h1, cuts[src], cuts[src + 1])
                if o:
                    out.append((src, dst, o[0], o[1]))
    return out


def source_from_mesh(mesh, first_point: int, first_stencil: int) -> SourceMesh:
    """SourceMesh view of a psn Mesh produced by psn_extract(PSN_EMIT) on a slab."""
    c = mesh.c
    return SourceMesh(first_point=first_point, n_points=c.n_points, halo_lo=c.halo_lo_points,
                      first_stencil=first_stencil, points=mesh.points, face_masks=mesh.face_masks[:c.n_points],
                      stencil_offsets=mesh.stencil_offsets[:c.n_points + 1], stencil_ids=mesh.stencil_ids[:c.n_stencil])


def shard_mesh(psn, shard: Shard):
    """A psn Mesh (window-indexed, as psn_smooth_prepare / psn_smooth_step expect) over a Shard."""
    from .psn import Mesh, MeshC
    dev = shard.points.device
    dummy = torch.zeros((1, 4), dtype=torch.int32, device=dev)
    m = Mesh(points=shard.points if shard.points.numel() else torch.zeros((1, 3), dtype=torch.float32, device=dev),
             quads=dummy, pairs=dummy[:, :2].contiguous(), stencil_offsets=shard.stencil_offsets,
             stencil_ids=shard.stencil_ids if shard.stencil_ids.numel() else torch.zeros(1, dtype=torch.int32, device=dev),
             face_masks=shard.face_masks if shard.face_masks.numel() else torch.zeros(1, dtype=torch.uint8, device=dev))
    c = MeshC()
    c.points = m.points.data_ptr(); c.quads = m.quads.data_ptr(); c.pairs = m.pairs.data_ptr()
    c.stencil_offsets = m.stencil_offsets.data_ptr(); c.stencil_ids = m.stencil_ids.data_ptr()
    c.face_masks = m.face_masks.data_ptr()
    c.cap_points = m.points.shape[0]; c.cap_quads = 1; c.cap_stencil = m.stencil_ids.shape[0]
    c.n_points, c.n_quads, c.n_stencil = shard.n_points, 0, shard.stencil_ids.numel()
    c.halo_lo_points, c.halo_hi_points = shard.halo_lo, shard.halo_hi
    c.first_point = shard.a0
    c.first_quad = 0
    c.first_stencil = (int(shard.stencil_offsets[0].item()) & 0xFFFFFFFF) if shard.n_points else 0
    m.c = c
    return m
