"""Sub-volume blocks stitched into the whole-volume mesh.

PAPER P:264 (open boundaries: sub-volumes add no artificial partitions) and
P:271 ("PSN can be employed in this manner [sub-volumes of a larger input
volume], with special attention placed on stitching output meshes together at
subvolume boundaries").  Marshalling only -- every step runs in libpsn.so:

    per block   psn_block_gather -> psn_extract (standalone box volume) -> psn_stitch_count
    once        psn_stitch_scan  (segment offsets; one read-back of the 3 totals)
    per block   psn_stitch_emit  (owned points / quads / stencils with whole-volume ids)

Only one block's box needs to be resident on the device at a time, and the
global label volume may live in host memory (pinned): the out-of-core use the
paper names.  The stitched mesh is bit-identical to ``PSN.extract`` over the
whole volume (tests/test_gpu_blocks.py).
"""
from __future__ import annotations

import ctypes

import torch

from .psn import PSN, Block, Mesh, MeshC, Volume, _DTYPES, _ptr, _stream


def block_cuts(n_vox: int, parts: int) -> list[int]:
    """Even cut points 0 = c_0 < c_1 < ... < c_p = n_vox of n_vox voxels into p = min(parts, n_vox) ranges."""
    p = max(1, min(int(parts), int(n_vox)))
    return [(n_vox * t) // p for t in range(p + 1)]


class BlockedExtractor:
    """Extract a label volume block by block and stitch the blocks into the whole-volume mesh.

    ``cuts``: per axis the voxel cut points (list of 3 lists, each starting at 0 and ending at the
    axis' voxel count), or ``blocks`` = (bx, by, bz) for even cuts.  ``keep_local``: keep every block's
    local mesh between the two passes (in-core); False re-gathers and re-extracts each block in the
    emit pass, so only one block is resident at a time (out-of-core).
    """

    def __init__(self, psn: PSN, dims, blocks=(2, 2, 1), cuts=None, spacing=(1.0, 1.0, 1.0),
                 origin=(0.0, 0.0, 0.0), label_set=None, keep_local: bool = True):
        self.psn = psn
        self.dims = tuple(int(d) for d in dims)
        if cuts is None:
            cuts = [block_cuts(self.dims[a] - 1, blocks[a]) for a in range(3)]
        self.cuts = [list(c) for c in cuts]
        for a in range(3):
            c = self.cuts[a]
            if c[0] != 0 or c[-1] != self.dims[a] - 1 or any(c[t] >= c[t + 1] for t in range(len(c) - 1)):
                raise ValueError(f"axis {a}: cuts must increase from 0 to {self.dims[a] - 1}")
        self.spacing, self.origin = tuple(spacing), tuple(origin)
        self.label_set = label_set
        self.keep_local = keep_local
        self.timings = None   # set to {} to collect per-phase CUDA-event times of the next run()
        self._events = []
        self.nxseg = len(self.cuts[0]) - 1
        self.nseg = (self.dims[1] - 1) * (self.dims[2] - 1) * self.nxseg
        self.blocks = []
        for c in range(len(self.cuts[2]) - 1):
            for b in range(len(self.cuts[1]) - 1):
                for a in range(self.nxseg):
                    blk = Block()
                    for d in range(3):
                        blk.dims[d] = self.dims[d]
                    lo = (self.cuts[0][a], self.cuts[1][b], self.cuts[2][c])
                    hi = (self.cuts[0][a + 1], self.cuts[1][b + 1], self.cuts[2][c + 1])
                    for d in range(3):
                        blk.own_lo[d], blk.own_hi[d] = lo[d], hi[d]
                    blk.xseg, blk.nxseg = a, self.nxseg
                    psn._check(psn.L.psn_block_box(ctypes.byref(blk), 0))
                    self.blocks.append(blk)

    def global_volume(self, dtype) -> Volume:
        """psn_volume of the whole volume for psn_stitch_emit / psn_smooth (labels unused: NULL)."""
        v = Volume()
        v.labels = None
        v.dtype = _DTYPES[dtype]
        for a in range(3):
            v.dims[a] = self.dims[a]; v.spacing[a] = float(self.spacing[a]); v.origin[a] = float(self.origin[a])
        v.z_lo, v.z_hi, v.own_k0, v.own_k1 = 0, self.dims[2], 0, self.dims[2] - 1
        return v

    def _mark(self, name):
        if self.timings is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self._events.append((name, ev))

    def _local(self, labels: torch.Tensor, blk: Block, stream):
        psn = self.psn
        shape = tuple(int(blk.box_hi[a] - blk.box_lo[a]) for a in (2, 1, 0))
        buf = torch.empty(shape, dtype=labels.dtype, device=f"cuda:{psn.device}")
        psn._check(psn.L.psn_block_gather(psn.h, ctypes.c_void_p(labels.data_ptr()), _DTYPES[labels.dtype],
                                          ctypes.byref(blk), _ptr(buf), _stream(stream)))
        self._mark("gather")
        vol = psn.volume(buf)                 # standalone: origin 0, spacing 1 (exact voxel centres)
        mesh = psn.extract(vol, self.label_set, stream=stream)
        self._mark("extract")
        n = ctypes.c_size_t()
        psn._check(psn.L.psn_stitch_workspace(ctypes.byref(blk), ctypes.byref(n)))
        sws = torch.empty(n.value, dtype=torch.uint8, device=buf.device)
        return mesh, sws

    def run(self, labels: torch.Tensor, stream=None) -> Mesh:
        """labels: (O, N, M) uint8/uint16/uint32, contiguous, CUDA or (pinned) CPU.  Returns the stitched
        whole-volume Mesh (``.c`` holds its totals, like PSN.extract's)."""
        psn = self.psn
        if labels.dtype not in _DTYPES or not labels.is_contiguous() or \
                tuple(labels.shape) != (self.dims[2], self.dims[1], self.dims[0]):
            raise ValueError("labels must be a contiguous (O, N, M) uint8/uint16/uint32 tensor")
        dev = f"cuda:{psn.device}"
        for blk in self.blocks:   # x rows of whole 16-byte units (TMA staging) where the volume allows
            psn._check(psn.L.psn_block_box(ctypes.byref(blk), _DTYPES[labels.dtype]))
        self._events = []
        self._mark("start")
        seg = torch.empty((3, self.nseg), dtype=torch.int32, device=dev)
        off = torch.empty_like(seg)
        totals = torch.empty(3, dtype=torch.int64, device=dev)
        kept = []
        for blk in self.blocks:   # pass 1: per-segment counts
            mesh, sws = self._local(labels, blk, stream)
            psn._check(psn.L.psn_stitch_count(psn.h, ctypes.byref(blk), ctypes.byref(mesh.c), _ptr(sws), sws.numel(),
                                              _ptr(seg), _stream(stream)))
            self._mark("stitch_count")
            kept.append((mesh, sws) if self.keep_local else None)
        nbytes = psn.L.psn_stitch_scan_workspace(self.nseg)
        scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        host = (ctypes.c_int64 * 3)()
        psn._check(psn.L.psn_stitch_scan(psn.h, self.nseg, _ptr(seg), _ptr(off), _ptr(totals), _ptr(scratch), nbytes,
                                         host, _stream(stream)))
        self._mark("stitch_scan")
        P, Q, S = int(host[0]), int(host[1]), int(host[2])
        out = psn.alloc_mesh(P, P, Q, S)
        c = MeshC()
        c.n_points, c.n_quads, c.n_stencil = P, Q, S
        psn._fill(out, c)
        gvol = self.global_volume(labels.dtype)
        for blk, k in zip(self.blocks, kept):   # pass 2: owned outputs with whole-volume ids
            if k is None:
                mesh, sws = self._local(labels, blk, stream)
                psn._check(psn.L.psn_stitch_count(psn.h, ctypes.byref(blk), ctypes.byref(mesh.c), _ptr(sws),
                                                  sws.numel(), None, _stream(stream)))
            else:
                mesh, sws = k
            psn._check(psn.L.psn_stitch_emit(psn.h, ctypes.byref(blk), ctypes.byref(gvol), ctypes.byref(mesh.c),
                                             _ptr(sws), sws.numel(), _ptr(off), _ptr(totals), ctypes.byref(out.c),
                                             _stream(stream)))
            self._mark("stitch_emit")
        out.volume = gvol
        if self.timings is not None:   # per-phase device time (ms), summed over blocks
            torch.cuda.synchronize()
            self.timings.clear()
            for (_, a), (name, b) in zip(self._events, self._events[1:]):
                self.timings[name] = self.timings.get(name, 0.0) + a.elapsed_time(b)
        return out
