"""Thin ctypes binding of the C ABI in include/psn.h (argument marshalling only).

Every step of the hot path runs in libpsn.so's sm_100a kernels; this module
only converts torch tensors to pointers and sizes, allocates output tensors
with the exact sizes the COUNT phase reports ("memory is
precisely allocated"), and raises on any non-OK status.  There is no CPU
fallback: if the extension or a CUDA device is missing, it raises.

Names follow include/psn.h: psn_extract / psn_smooth / psn_triangulate.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PSN_LIB") or os.path.join(_HERE, "libpsn.so")   # PSN_LIB: A/B builds (tools)

PSN_OK, PSN_ERR_ARG, PSN_ERR_LABELS, PSN_ERR_OVERFLOW, PSN_ERR_CAPACITY, PSN_ERR_STATE, PSN_ERR_CUDA = range(7)
PSN_COUNT, PSN_EMIT, PSN_DEVICE = 1, 2, 4
PSN_TRI_FIXED_02, PSN_TRI_SHORTEST, PSN_TRI_MIN_AREA, PSN_TRI_MOST_COPLANAR = 0, 1, 2, 3
PSN_CONSTRAINT_BOX, PSN_CONSTRAINT_SPHERE = 0, 1
BACKGROUND = 0xFFFFFFFF

_DTYPES = {torch.uint8: 1, torch.uint16: 2, torch.uint32: 4}


class PSNError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "PSN_OK", 1: "PSN_ERR_ARG", 2: "PSN_ERR_LABELS", 3: "PSN_ERR_OVERFLOW",
           4: "PSN_ERR_CAPACITY", 5: "PSN_ERR_STATE", 6: "PSN_ERR_CUDA"}


class Volume(ctypes.Structure):
    _fields_ = [("labels", ctypes.c_void_p), ("dtype", ctypes.c_int), ("dims", ctypes.c_int64 * 3),
                ("spacing", ctypes.c_double * 3), ("origin", ctypes.c_double * 3),
                ("z_lo", ctypes.c_int64), ("z_hi", ctypes.c_int64),
                ("own_k0", ctypes.c_int64), ("own_k1", ctypes.c_int64)]


class Labels(ctypes.Structure):
    _fields_ = [("values", ctypes.POINTER(ctypes.c_uint32)), ("count", ctypes.c_int64), ("all_nonzero", ctypes.c_int)]


class MeshC(ctypes.Structure):
    _fields_ = [("points", ctypes.c_void_p), ("quads", ctypes.c_void_p), ("pairs", ctypes.c_void_p),
                ("stencil_offsets", ctypes.c_void_p), ("stencil_ids", ctypes.c_void_p),
                ("face_masks", ctypes.c_void_p),
                ("cap_points", ctypes.c_int64), ("cap_quads", ctypes.c_int64), ("cap_stencil", ctypes.c_int64),
                ("n_points", ctypes.c_int64), ("n_quads", ctypes.c_int64), ("n_stencil", ctypes.c_int64),
                ("halo_lo_points", ctypes.c_int64), ("halo_hi_points", ctypes.c_int64),
                ("first_point", ctypes.c_int64), ("first_quad", ctypes.c_int64), ("first_stencil", ctypes.c_int64),
                ("smooth_cache", ctypes.c_void_p), ("smooth_cache_valid", ctypes.c_int64),
                ("first_dev", ctypes.c_void_p)]


class Block(ctypes.Structure):
    _fields_ = [("dims", ctypes.c_int64 * 3), ("own_lo", ctypes.c_int64 * 3), ("own_hi", ctypes.c_int64 * 3),
                ("box_lo", ctypes.c_int64 * 3), ("box_hi", ctypes.c_int64 * 3), ("xseg", ctypes.c_int64),
                ("nxseg", ctypes.c_int64)]


class IpcHandle(ctypes.Structure):
    _fields_ = [("handle", ctypes.c_ubyte * 64), ("offset", ctypes.c_uint64)]


class PeerSide(ctypes.Structure):
    _fields_ = [("dst", ctypes.c_void_p * 2), ("src_begin", ctypes.c_int64), ("src_end", ctypes.c_int64),
                ("dst_begin", ctypes.c_int64), ("peer_sig", ctypes.c_void_p)]


class Peer(ctypes.Structure):
    _fields_ = [("side", PeerSide * 2), ("sig", ctypes.c_void_p), ("ctr", ctypes.c_void_p), ("err", ctypes.c_void_p),
                ("ctr_base", ctypes.c_uint64), ("iteration", ctypes.c_uint64)]


_lib = None


def lib():
    """Load libpsn.so (build it with __graft_entry__.build()); raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libpsn.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        L.psn_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
        L.psn_ctx_create.restype = ctypes.c_int
        L.psn_ctx_destroy.argtypes = [vp]
        L.psn_ctx_destroy.restype = None
        L.psn_last_error.argtypes = [vp]
        L.psn_last_error.restype = ctypes.c_char_p
        L.psn_status_string.argtypes = [ctypes.c_int]
        L.psn_status_string.restype = ctypes.c_char_p
        L.psn_extract_workspace.argtypes = [ctypes.POINTER(Volume), ctypes.POINTER(ctypes.c_size_t)]
        L.psn_extract_workspace.restype = ctypes.c_int
        L.psn_extract.argtypes = [vp, ctypes.POINTER(Volume), ctypes.POINTER(Labels), ctypes.POINTER(MeshC),
                                  ctypes.c_uint, vp, ctypes.c_size_t, vp]
        L.psn_extract.restype = ctypes.c_int
        L.psn_extract_totals.argtypes = [vp, ctypes.POINTER(Volume), vp, ctypes.c_size_t, vp, vp]
        L.psn_extract_totals.restype = ctypes.c_int
        L.psn_mesh_totals.argtypes = [vp, ctypes.POINTER(Volume), ctypes.POINTER(MeshC), vp, ctypes.c_size_t, vp]
        L.psn_mesh_totals.restype = ctypes.c_int
        L.psn_extract_rows.argtypes = [vp, ctypes.POINTER(Volume), vp, ctypes.c_size_t, vp, vp,
                                       ctypes.POINTER(ctypes.c_int64), vp]
        L.psn_extract_rows.restype = ctypes.c_int
        L.psn_smooth_workspace.argtypes = [ctypes.POINTER(MeshC), ctypes.POINTER(ctypes.c_size_t)]
        L.psn_smooth_workspace.restype = ctypes.c_int
        L.psn_smooth_prepare.argtypes = [vp, ctypes.POINTER(Volume), ctypes.POINTER(MeshC), vp, ctypes.c_size_t, vp]
        L.psn_smooth_prepare.restype = ctypes.c_int
        L.psn_smooth.argtypes = [vp, ctypes.POINTER(Volume), ctypes.POINTER(MeshC), vp, ctypes.c_int32,
                                 ctypes.c_float, ctypes.c_float, vp, ctypes.c_size_t, vp]
        L.psn_smooth.restype = ctypes.c_int
        L.psn_smooth_step.argtypes = [vp, ctypes.POINTER(Volume), ctypes.POINTER(MeshC), vp, ctypes.c_size_t, vp, vp,
                                      ctypes.c_float, ctypes.c_float, vp]
        L.psn_smooth_step.restype = ctypes.c_int
        L.psn_smooth_finalize.argtypes = [vp, ctypes.POINTER(Volume), ctypes.POINTER(MeshC), vp, i64, i64, vp, vp]
        L.psn_smooth_finalize.restype = ctypes.c_int
        L.psn_triangulate.argtypes = [vp, ctypes.POINTER(MeshC), vp, ctypes.c_int, vp, vp]
        L.psn_triangulate.restype = ctypes.c_int
        L.psn_ctx_set_smoothing.argtypes = [vp, ctypes.c_int, ctypes.c_int32, ctypes.c_int32]
        L.psn_ctx_set_smoothing.restype = ctypes.c_int
        if hasattr(L, "psn_ctx_set_constraint"):   # (absent from older builds loaded via PSN_LIB)
            L.psn_ctx_set_constraint.argtypes = [vp, ctypes.c_int]
            L.psn_ctx_set_constraint.restype = ctypes.c_int
        L.psn_ctx_set_emission.argtypes = [vp, ctypes.c_int]
        L.psn_ctx_set_emission.restype = ctypes.c_int
        L.psn_ctx_set_counting.argtypes = [vp, ctypes.c_int]
        L.psn_ctx_set_counting.restype = ctypes.c_int
        L.psn_smooth_status.argtypes = [vp, ctypes.POINTER(MeshC), vp, ctypes.c_size_t, vp]
        L.psn_smooth_status.restype = ctypes.c_int
        L.psn_ctx_set_smooth_events.argtypes = [vp, ctypes.POINTER(vp)]
        L.psn_ctx_set_smooth_events.restype = ctypes.c_int
        L.psn_ctx_set_pass_events.argtypes = [vp, ctypes.POINTER(vp)]
        L.psn_ctx_set_pass_events.restype = ctypes.c_int
        L.psn_launch_count.argtypes = [vp]
        L.psn_launch_count.restype = i64
        if hasattr(L, "psn_smooth_step_peer"):   # (absent from older builds loaded via PSN_LIB)
            L.psn_smooth_step_peer.argtypes = [vp, ctypes.POINTER(Volume), ctypes.POINTER(MeshC), vp, ctypes.c_size_t,
                                               vp, vp, ctypes.c_int, ctypes.c_float, ctypes.c_float,
                                               ctypes.POINTER(Peer), vp]
            L.psn_smooth_step_peer.restype = ctypes.c_int
            L.psn_smooth_run_peer.argtypes = [vp, ctypes.POINTER(Volume), ctypes.POINTER(MeshC), vp, ctypes.c_size_t,
                                              vp, vp, ctypes.c_int32, ctypes.c_float, ctypes.c_float,
                                              ctypes.POINTER(Peer), vp]
            L.psn_smooth_run_peer.restype = ctypes.c_int
            L.psn_ipc_export.argtypes = [vp, vp, ctypes.POINTER(IpcHandle)]
            L.psn_ipc_export.restype = ctypes.c_int
            L.psn_ipc_open.argtypes = [vp, ctypes.POINTER(IpcHandle), ctypes.POINTER(vp)]
            L.psn_ipc_open.restype = ctypes.c_int
            L.psn_ipc_close.argtypes = [vp, vp]
            L.psn_ipc_close.restype = ctypes.c_int
        if hasattr(L, "psn_stitch_emit"):   # (absent from older builds loaded via PSN_LIB)
            BP = ctypes.POINTER(Block)
            L.psn_block_box.argtypes = [BP, ctypes.c_int]
            L.psn_block_box.restype = ctypes.c_int
            L.psn_block_gather.argtypes = [vp, vp, ctypes.c_int, BP, vp, vp]
            L.psn_block_gather.restype = ctypes.c_int
            L.psn_stitch_workspace.argtypes = [BP, ctypes.POINTER(ctypes.c_size_t)]
            L.psn_stitch_workspace.restype = ctypes.c_int
            L.psn_stitch_count.argtypes = [vp, BP, ctypes.POINTER(MeshC), vp, ctypes.c_size_t, vp, vp]
            L.psn_stitch_count.restype = ctypes.c_int
            L.psn_stitch_scan_workspace.argtypes = [i64]
            L.psn_stitch_scan_workspace.restype = ctypes.c_size_t
            L.psn_stitch_scan.argtypes = [vp, i64, vp, vp, vp, vp, ctypes.c_size_t, ctypes.POINTER(ctypes.c_int64), vp]
            L.psn_stitch_scan.restype = ctypes.c_int
            L.psn_stitch_emit.argtypes = [vp, BP, ctypes.POINTER(Volume), ctypes.POINTER(MeshC), vp, ctypes.c_size_t,
                                          vp, vp, ctypes.POINTER(MeshC), vp]
            L.psn_stitch_emit.restype = ctypes.c_int
        _lib = L
    return _lib


EXPORTED = ["psn_ctx_create", "psn_ctx_destroy", "psn_last_error", "psn_status_string",
            "psn_extract_workspace", "psn_extract", "psn_extract_rows", "psn_extract_totals", "psn_mesh_totals", "psn_smooth_workspace",
            "psn_smooth_prepare", "psn_smooth", "psn_smooth_step", "psn_smooth_finalize", "psn_triangulate", "psn_launch_count",
            "psn_ctx_set_smoothing", "psn_ctx_set_pass_events", "psn_ctx_set_smooth_events", "psn_smooth_status", "psn_ctx_set_counting",
            "psn_ctx_set_emission", "psn_ctx_set_constraint", "psn_smooth_step_peer", "psn_smooth_run_peer", "psn_ipc_export",
            "psn_ipc_open", "psn_ipc_close", "psn_block_box", "psn_block_gather", "psn_stitch_workspace",
            "psn_stitch_count", "psn_stitch_scan_workspace", "psn_stitch_scan", "psn_stitch_emit"]


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


@dataclass
class Mesh:
    """Device mesh (window-indexed points, own-point stencils, own quads)."""
    points: torch.Tensor          # float32 [halo_lo + P + halo_hi, 3]
    quads: torch.Tensor           # uint32 [Q, 4] (stored as int32 view)
    pairs: torch.Tensor           # uint32 [Q, 2]
    stencil_offsets: torch.Tensor  # uint32 [P + 1]
    stencil_ids: torch.Tensor     # uint32 [S]
    face_masks: torch.Tensor      # uint8 [P]
    smooth_cache: torch.Tensor | None = None   # uint32 [W, 2] packed smoothing cache (written by PSN_EMIT)
    c: MeshC = field(default_factory=MeshC)

    @property
    def n_points(self):
        return self.c.n_points

    @property
    def n_quads(self):
        return self.c.n_quads

    @property
    def n_stencil(self):
        return self.c.n_stencil

    @property
    def n_window(self):
        return self.c.halo_lo_points + self.c.n_points + self.c.halo_hi_points


class PSN:
    """One context per device (psn_ctx)."""

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("PSN needs a CUDA device (no CPU fallback)")
        self.L = lib()
        self.device = device
        h = ctypes.c_void_p()
        rc = self.L.psn_ctx_create(device, ctypes.byref(h))
        if rc != PSN_OK:
            raise PSNError(rc, "psn_ctx_create failed")
        self.h = h
        self._ws = {}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.L.psn_ctx_destroy(self.h)
        except Exception:
            pass

    def _check(self, rc):
        if rc != PSN_OK:
            raise PSNError(rc, self.L.psn_last_error(self.h).decode())

    @property
    def launches(self):
        return self.L.psn_launch_count(self.h)

    # ------------------------------------------------------------------ volume / labels
    @staticmethod
    def volume(labels: torch.Tensor, dims=None, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0),
               z_lo: int = 0, own=None) -> Volume:
        if labels.dtype not in _DTYPES or not labels.is_cuda or not labels.is_contiguous():
            raise ValueError("labels must be a contiguous CUDA uint8/uint16/uint32 tensor (z, y, x)")
        Z, N, M = labels.shape
        if dims is None:
            dims = (M, N, Z)
        v = Volume()
        v.labels = labels.data_ptr()
        v._keep = labels   # the struct holds a raw device pointer: keep the tensor alive with it
        v.dtype = _DTYPES[labels.dtype]
        for a in range(3):
            v.dims[a] = int(dims[a]); v.spacing[a] = float(spacing[a]); v.origin[a] = float(origin[a])
        v.z_lo, v.z_hi = z_lo, z_lo + Z
        k0, k1 = own if own is not None else (0, dims[2] - 1)
        v.own_k0, v.own_k1 = int(k0), int(k1)
        return v

    @staticmethod
    def labels(label_set=None):
        lab = Labels()
        if label_set is None:
            lab.all_nonzero = 1
            lab.count = 0
            lab._keep = None
        else:
            vals = list(label_set)
            arr = (ctypes.c_uint32 * max(len(vals), 1))(*vals)
            lab.values = ctypes.cast(arr, ctypes.POINTER(ctypes.c_uint32))
            lab.count = len(vals)
            lab.all_nonzero = 0
            lab._keep = arr
        return lab

    def workspace(self, vol: Volume) -> torch.Tensor:
        n = ctypes.c_size_t()
        rc = self.L.psn_extract_workspace(ctypes.byref(vol), ctypes.byref(n))
        self._check(rc)
        return torch.empty(n.value, dtype=torch.uint8, device=f"cuda:{self.device}")

    # ------------------------------------------------------------------ extraction
    def count(self, vol: Volume, labels: Labels, ws: torch.Tensor, stream=None) -> MeshC:
        """psn_extract(PSN_COUNT): totals (one stream synchronisation)."""
        m = MeshC()
        rc = self.L.psn_extract(self.h, ctypes.byref(vol), ctypes.byref(labels), ctypes.byref(m), PSN_COUNT,
                                _ptr(ws), ws.numel(), _stream(stream))
        self._check(rc)
        return m

    def count_device(self, vol: Volume, labels: Labels, ws: torch.Tensor, totals: torch.Tensor, stream=None):
        """psn_extract(PSN_COUNT|PSN_DEVICE) + psn_extract_totals: no host round trip; `totals` (device int64[5])
        receives (P, Q, S, halo_lo, halo_hi) of this call."""
        m = MeshC()
        self._check(self.L.psn_extract(self.h, ctypes.byref(vol), ctypes.byref(labels), ctypes.byref(m),
                                       PSN_COUNT | PSN_DEVICE, _ptr(ws), ws.numel(), _stream(stream)))
        self._check(self.L.psn_extract_totals(self.h, ctypes.byref(vol), _ptr(ws), ws.numel(), _ptr(totals),
                                              _stream(stream)))

    def emit_device(self, vol: Volume, labels: Labels, ws: torch.Tensor, mesh: "Mesh", first_dev: torch.Tensor,
                    stream=None):
        """psn_extract(PSN_EMIT|PSN_DEVICE) into `mesh` (its capacities and host fields from an earlier
        count of the same volume) with the global first ids from device int64[3] `first_dev`."""
        c = MeshC.from_buffer_copy(mesh.c)
        self._fill(mesh, c, (c.first_point, c.first_quad, c.first_stencil))
        mesh.c.first_dev = first_dev.data_ptr()
        rc = self.L.psn_extract(self.h, ctypes.byref(vol), ctypes.byref(labels), ctypes.byref(mesh.c),
                                PSN_EMIT | PSN_DEVICE, _ptr(ws), ws.numel(), _stream(stream))
        mesh.c.first_dev = None
        self._check(rc)

    def alloc_mesh(self, n_window, n_points, n_quads, n_stencil, smooth_cache: bool = False) -> Mesh:
        """Exactly sized output arrays; smooth_cache=True adds the packed smoothing cache the
        emission can write (psn_mesh.smooth_cache): psn_smooth then skips its prep pass --
        8 more bytes per point written by the emission instead of ~29 read + 8 written by
        k_smooth_prep8 (measured: c4 step -1 %, but extraction +2 %, c5a extraction +13 %)."""
        dev = f"cuda:{self.device}"
        return Mesh(points=torch.empty((max(n_window, 1), 3), dtype=torch.float32, device=dev),
                    quads=torch.empty((max(n_quads, 1), 4), dtype=torch.int32, device=dev),
                    pairs=torch.empty((max(n_quads, 1), 2), dtype=torch.int32, device=dev),
                    stencil_offsets=torch.empty(n_points + 1, dtype=torch.int32, device=dev),
                    stencil_ids=torch.empty(max(n_stencil, 1), dtype=torch.int32, device=dev),
                    face_masks=torch.empty(max(n_points, 1), dtype=torch.uint8, device=dev),
                    smooth_cache=torch.empty((max(n_window, 1), 2), dtype=torch.int32, device=dev)
                    if smooth_cache else None)

    def _fill(self, mesh: Mesh, c: MeshC, first=(0, 0, 0)):
        c.points = mesh.points.data_ptr(); c.quads = mesh.quads.data_ptr(); c.pairs = mesh.pairs.data_ptr()
        c.stencil_offsets = mesh.stencil_offsets.data_ptr(); c.stencil_ids = mesh.stencil_ids.data_ptr()
        c.face_masks = mesh.face_masks.data_ptr()
        c.smooth_cache = mesh.smooth_cache.data_ptr() if mesh.smooth_cache is not None else None
        c.smooth_cache_valid = 0
        c.cap_points = mesh.points.shape[0]; c.cap_quads = mesh.quads.shape[0]; c.cap_stencil = mesh.stencil_ids.shape[0]
        c.first_point, c.first_quad, c.first_stencil = (int(x) for x in first)
        mesh.c = c

    def emit(self, vol: Volume, labels: Labels, ws: torch.Tensor, counted: MeshC, first=(0, 0, 0),
             mesh: Mesh | None = None, stream=None) -> Mesh:
        """psn_extract(PSN_EMIT) into exactly allocated arrays."""
        if mesh is None:
            mesh = self.alloc_mesh(counted.halo_lo_points + counted.n_points + counted.halo_hi_points,
                                   counted.n_points, counted.n_quads, counted.n_stencil)
        c = MeshC.from_buffer_copy(counted)
        self._fill(mesh, c, first)
        rc = self.L.psn_extract(self.h, ctypes.byref(vol), ctypes.byref(labels), ctypes.byref(mesh.c), PSN_EMIT,
                                _ptr(ws), ws.numel(), _stream(stream))
        self._check(rc)
        return mesh

    def extract(self, vol: Volume, label_set=None, ws=None, stream=None) -> Mesh:
        """Two-phase extraction: COUNT (exact totals) -> allocate -> EMIT."""
        labels = self.labels(label_set)
        if ws is None:
            ws = self.workspace(vol)
        counted = self.count(vol, labels, ws, stream)
        mesh = self.emit(vol, labels, ws, counted, stream=stream)
        mesh.ws = ws
        return mesh

    def extract_into(self, vol: Volume, labels: Labels, ws: torch.Tensor, mesh: Mesh, stream=None) -> None:
        """Steady state: PSN_COUNT|PSN_EMIT with preallocated capacities, no host sync."""
        c = MeshC()
        self._fill(mesh, c)
        rc = self.L.psn_extract(self.h, ctypes.byref(vol), ctypes.byref(labels), ctypes.byref(mesh.c),
                                PSN_COUNT | PSN_EMIT, _ptr(ws), ws.numel(), _stream(stream))
        self._check(rc)

    def totals(self, vol: Volume, ws: torch.Tensor, mesh: Mesh, stream=None) -> Mesh:
        rc = self.L.psn_mesh_totals(self.h, ctypes.byref(vol), ctypes.byref(mesh.c), _ptr(ws), ws.numel(),
                                    _stream(stream))
        self._check(rc)
        return mesh

    def rows(self, vol: Volume, ws: torch.Tensor, stream=None):
        """psn_extract_rows: per voxel row (counts int32 [3, R] = P/Q/S, trims int32 [R, 2] = [xL, xR))
        of the last PSN_COUNT on ws (uint32 values in int32 tensors)."""
        R = ctypes.c_int64()
        self._check(self.L.psn_extract_rows(self.h, ctypes.byref(vol), _ptr(ws), ws.numel(), None, None,
                                            ctypes.byref(R), _stream(stream)))
        dev = ws.device
        counts = torch.empty((3, max(R.value, 1)), dtype=torch.int32, device=dev)
        trims = torch.empty((max(R.value, 1), 2), dtype=torch.int32, device=dev)
        self._check(self.L.psn_extract_rows(self.h, ctypes.byref(vol), _ptr(ws), ws.numel(), _ptr(counts),
                                            _ptr(trims), None, _stream(stream)))
        return counts[:, :R.value], trims[:R.value]

    # ------------------------------------------------------------------ smoothing / triangulation
    def smooth_workspace(self, mesh: Mesh) -> torch.Tensor:
        n = ctypes.c_size_t()
        self._check(self.L.psn_smooth_workspace(ctypes.byref(mesh.c), ctypes.byref(n)))
        return torch.empty(max(n.value, 1), dtype=torch.uint8, device=f"cuda:{self.device}")

    def smooth(self, vol: Volume, mesh: Mesh, iterations: int, relaxation: float, constraint: float,
               out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty((max(mesh.n_window, 1), 3), dtype=torch.float32, device=mesh.points.device)
        if ws is None:
            ws = self.smooth_workspace(mesh)
        rc = self.L.psn_smooth(self.h, ctypes.byref(vol), ctypes.byref(mesh.c), _ptr(out), int(iterations),
                               float(relaxation), float(constraint), _ptr(ws), ws.numel(), _stream(stream))
        self._check(rc)
        return out

    def set_smoothing(self, mode: int = 1, iterations_per_launch: int = 0, points_per_tile: int = 0):
        """1 = one launch per iteration (default), 0 = wavefront (temporally blocked)."""
        self._check(self.L.psn_ctx_set_smoothing(self.h, int(mode), int(iterations_per_launch), int(points_per_tile)))

    def set_pass_events(self, events=None):
        """Record 4 torch.cuda.Events around the passes of every later psn_extract (None: stop):
        [0] before counting, [1] counting -> scan, [2] scan -> emission, [3] after emission."""
        if events is None:
            self._check(self.L.psn_ctx_set_pass_events(self.h, None))
            self._pass_events = None
            return
        assert len(events) == 4
        for e in events:   # torch creates the CUDA event lazily: force it (once)
            if not e.cuda_event:
                e.record()
        arr = (ctypes.c_void_p * 4)(*[ctypes.c_void_p(e.cuda_event) for e in events])
        self._pass_events = (events, arr)
        self._check(self.L.psn_ctx_set_pass_events(self.h, arr))

    def set_smooth_events(self, events=None):
        """Record 2 torch.cuda.Events around the Jacobi launches of every later psn_smooth (None: stop)."""
        if events is None:
            self._check(self.L.psn_ctx_set_smooth_events(self.h, None))
            self._smooth_events = None
            return
        assert len(events) == 2
        for e in events:
            if not e.cuda_event:
                e.record()
        arr = (ctypes.c_void_p * 2)(*[ctypes.c_void_p(e.cuda_event) for e in events])
        self._smooth_events = (events, arr)
        self._check(self.L.psn_ctx_set_smooth_events(self.h, arr))

    def set_counting(self, mode: int = 0):
        """0 = automatic (warp-per-row k_count3 when a row fits a warp), 1 = x-tiled k_count."""
        self._check(self.L.psn_ctx_set_counting(self.h, int(mode)))

    def set_constraint(self, shape: int = PSN_CONSTRAINT_BOX):
        """Motion constraint of psn_smooth: box (per axis, default) or sphere (radius d*min(s))."""
        self._check(self.L.psn_ctx_set_constraint(self.h, int(shape)))

    def set_emission(self, mode: int = 0):
        """0 = automatic (band-staged k_emit_band), 2 = general scan-based k_emit."""
        self._check(self.L.psn_ctx_set_emission(self.h, int(mode)))

    def smooth_status(self, mesh: Mesh, ws: torch.Tensor, stream=None):
        self._check(self.L.psn_smooth_status(self.h, ctypes.byref(mesh.c), _ptr(ws), ws.numel(), _stream(stream)))

    def smooth_prepare(self, vol: Volume, mesh: Mesh, ws: torch.Tensor, stream=None):
        self._check(self.L.psn_smooth_prepare(self.h, ctypes.byref(vol), ctypes.byref(mesh.c), _ptr(ws), ws.numel(),
                                              _stream(stream)))

    @staticmethod
    def offsets_buffer(n_window: int, device) -> torch.Tensor:
        """A window offset buffer as psn_smooth_step reads / writes it: float32 [n_window][4]."""
        return torch.zeros((max(n_window, 1), 4), dtype=torch.float32, device=device)

    def smooth_step(self, vol: Volume, mesh: Mesh, ws: torch.Tensor, src: torch.Tensor | None, dst: torch.Tensor,
                    relaxation: float, constraint: float, stream=None):
        """One Jacobi step: src / dst are float32 [n_window][4] (x, y, z, unused) offset buffers."""
        rc = self.L.psn_smooth_step(self.h, ctypes.byref(vol), ctypes.byref(mesh.c), _ptr(ws), ws.numel(), _ptr(src),
                                    _ptr(dst), float(relaxation), float(constraint), _stream(stream))
        self._check(rc)

    def smooth_step_peer(self, vol: Volume, mesh: Mesh, ws: torch.Tensor, src: torch.Tensor | None,
                         dst: torch.Tensor, parity: int, relaxation: float, constraint: float, peer: "Peer",
                         stream=None):
        """psn_smooth_step + the peer halo push / signal (see psn.h); `peer` is advanced in place."""
        rc = self.L.psn_smooth_step_peer(self.h, ctypes.byref(vol), ctypes.byref(mesh.c), _ptr(ws), ws.numel(),
                                         _ptr(src), _ptr(dst), int(parity), float(relaxation), float(constraint),
                                         ctypes.byref(peer), _stream(stream))
        self._check(rc)

    def smooth_run_peer(self, vol: Volume, mesh: Mesh, ws: torch.Tensor, bufs, iterations: int, relaxation: float,
                        constraint: float, peer: "Peer", stream=None) -> torch.Tensor:
        """`iterations` peer steps in one call (bufs = two float4 window buffers); returns the final buffer."""
        rc = self.L.psn_smooth_run_peer(self.h, ctypes.byref(vol), ctypes.byref(mesh.c), _ptr(ws), ws.numel(),
                                        _ptr(bufs[0]), _ptr(bufs[1]), int(iterations), float(relaxation),
                                        float(constraint), ctypes.byref(peer), _stream(stream))
        self._check(rc)
        return bufs[(peer.iteration - 1) & 1] if iterations else None

    def ipc_export(self, t: torch.Tensor) -> bytes:
        """CUDA IPC handle (+ offset) of tensor t's memory, as bytes for the peer processes."""
        h = IpcHandle()
        self._check(self.L.psn_ipc_export(self.h, _ptr(t), ctypes.byref(h)))
        return bytes(h)

    def ipc_open(self, blob: bytes) -> int:
        """Map a peer's exported memory; returns the device address (int)."""
        h = IpcHandle.from_buffer_copy(blob)
        p = ctypes.c_void_p()
        self._check(self.L.psn_ipc_open(self.h, ctypes.byref(h), ctypes.byref(p)))
        return int(p.value)

    def ipc_close(self, addr: int):
        self._check(self.L.psn_ipc_close(self.h, ctypes.c_void_p(addr)))

    def smooth_finalize(self, vol: Volume, mesh: Mesh, offsets: torch.Tensor | None, out: torch.Tensor,
                        w0: int = 0, w1: int | None = None, stream=None):
        w1 = mesh.n_window if w1 is None else w1
        rc = self.L.psn_smooth_finalize(self.h, ctypes.byref(vol), ctypes.byref(mesh.c), _ptr(offsets), int(w0),
                                        int(w1), _ptr(out), _stream(stream))
        self._check(rc)
        return out

    def triangulate(self, mesh: Mesh, points: torch.Tensor, strategy: int = PSN_TRI_SHORTEST,
                    out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty((max(2 * mesh.n_quads, 1), 3), dtype=torch.int32, device=mesh.points.device)
        rc = self.L.psn_triangulate(self.h, ctypes.byref(mesh.c), _ptr(points), int(strategy), _ptr(out),
                                    _stream(stream))
        self._check(rc)
        return out


def to_numpy_u32(t: torch.Tensor, n_rows: int):
    """Device int32 view -> host numpy uint32 (first n_rows rows)."""
    return t[:n_rows].cpu().numpy().view("uint32")


class Pipeline:
    """Steady-state extract + smooth (+ triangulate) on one resident volume.

    Buffers are sized once from a two-phase warm-up extraction (COUNT ->
    allocate -> EMIT); every later run() is PSN_COUNT|PSN_EMIT with those
    capacities (no host synchronisation) followed by psn_smooth.
    """

    def __init__(self, psn: PSN, vol: Volume, iterations: int, relaxation: float, constraint: float,
                 label_set=None, triangulate: bool = False, headroom: float = 0.0, smooth_cache: bool = False):
        self.psn, self.vol = psn, vol
        self.T, self.lam, self.d = iterations, relaxation, constraint
        self.labels = psn.labels(label_set)
        self.ws = psn.workspace(vol)
        m0 = psn.extract(vol, label_set, ws=self.ws)
        self.counts = (m0.n_points, m0.n_quads, m0.n_stencil)
        h = 1.0 + headroom
        self.mesh = psn.alloc_mesh(int(m0.n_window * h) + 1, int(m0.n_points * h) + 1,
                                   int(m0.n_quads * h) + 1, int(m0.n_stencil * h) + 1, smooth_cache=smooth_cache)
        self.mesh.c = MeshC.from_buffer_copy(m0.c)
        self.sws = psn.smooth_workspace(self.mesh)
        self.out = torch.empty_like(self.mesh.points)
        self.tris = torch.empty((max(2 * self.mesh.quads.shape[0], 1), 3), dtype=torch.int32,
                                device=self.out.device) if triangulate else None
        self.launches = {}

    def extract(self, stream=None):
        self.psn.extract_into(self.vol, self.labels, self.ws, self.mesh, stream)
        # the totals are those of the warm-up volume (same volume every run)
        self.mesh.c.n_points, self.mesh.c.n_quads, self.mesh.c.n_stencil = self.counts
        self.launches["extract"] = self.psn.launches

    def smooth(self, stream=None):
        self.psn.smooth(self.vol, self.mesh, self.T, self.lam, self.d, out=self.out, ws=self.sws, stream=stream)
        self.launches["smooth"] = self.psn.launches
        if self.tris is not None:
            self.psn.triangulate(self.mesh, self.out, out=self.tris, stream=stream)
            self.launches["triangulate"] = self.psn.launches

    def run(self, stream=None):
        self.extract(stream)
        self.smooth(stream)

    def capture(self):
        """Capture the steady-state step into two CUDA graphs (extraction, smoothing [+ triangulation]):
        replay() then issues each with one launch instead of the library's per-kernel host calls --
        what bounds the small configs (c1, c2, c5b), whose kernels are shorter than their launch
        path.  Same kernels, same arguments, same outputs (tested).  Call after one run()."""
        torch.cuda.synchronize()
        self.g_ext, self.g_sm = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g_ext):
            self.extract()
        with torch.cuda.graph(self.g_sm):
            self.smooth()
        torch.cuda.synchronize()
        return self

    def replay_extract(self):
        self.g_ext.replay()

    def replay_smooth(self):
        self.g_sm.replay()

    def check(self, stream=None):
        """Synchronising read of the device totals / status of the last run."""
        self.psn.totals(self.vol, self.ws, self.mesh, stream)
        return (self.mesh.n_points, self.mesh.n_quads, self.mesh.n_stencil) == self.counts


def surface_nets_host(psn: PSN, labels_host: torch.Tensor, spacing, iterations: int, relaxation: float,
                      constraint: float, origin=(0.0, 0.0, 0.0), label_set=None, state: dict | None = None,
                      stream=None):
    """Public end-to-end call with HOST buffers: H2D copy of the label volume
    (pinned host tensor), extraction + smoothing on the device, D2H copy of the
    smoothed points, quads and two-tuples into pinned host tensors.  `state`
    caches device buffers across calls (pass the same dict each time)."""
    state = {} if state is None else state
    dev = f"cuda:{psn.device}"
    if "labels" not in state:
        state["labels"] = torch.empty(labels_host.shape, dtype=labels_host.dtype, device=dev)
    lab = state["labels"]
    lab.copy_(labels_host, non_blocking=True)
    vol = psn.volume(lab, spacing=spacing, origin=origin)
    if "pipe" not in state:
        state["pipe"] = Pipeline(psn, vol, iterations, relaxation, constraint, label_set)
        pipe = state["pipe"]
        P, Q = pipe.counts[0], pipe.counts[1]
        state["h_points"] = torch.empty((P, 3), dtype=torch.float32, pin_memory=True)
        state["h_quads"] = torch.empty((Q, 4), dtype=torch.int32, pin_memory=True)
        state["h_pairs"] = torch.empty((Q, 2), dtype=torch.int32, pin_memory=True)
    pipe = state["pipe"]
    pipe.vol = vol
    pipe.run(stream)
    P, Q = pipe.counts[0], pipe.counts[1]
    state["h_points"].copy_(pipe.out[:P], non_blocking=True)
    state["h_quads"].copy_(pipe.mesh.quads[:Q], non_blocking=True)
    state["h_pairs"].copy_(pipe.mesh.pairs[:Q], non_blocking=True)
    state["h2d_bytes"] = labels_host.numel() * labels_host.element_size()
    state["d2h_bytes"] = P * 12 + Q * 24
    return state["h_points"], state["h_quads"], state["h_pairs"]


class SurfaceNetsStream:
    """Pipelined host-buffer API for a sequence of same-shaped label volumes
    (e.g. a time series of segmentations, or an atlas re-extracted with new
    labels).

    submit(labels_host) enqueues, for one pinned host volume:
      copy stream    : host -> device copy of the labels (after the slot's
                       previous volume has been processed);
      compute stream : PSN_COUNT (one host synchronisation for the exact totals,
                       P:86), PSN_EMIT into the slot's mesh (grown if needed),
                       psn_smooth;
      readback stream: device -> pinned host copies of the quads and two-tuples
                       (as soon as extraction is done, overlapping smoothing) and
                       of the smoothed points.
    `depth` slots (device labels, workspaces, mesh, smoothing buffers, pinned
    host outputs) rotate, so volume s+1's upload overlaps volume s's compute and
    readback (PCIe is full duplex); a volume's compute is issued by the NEXT
    submit() (or result() / flush()), after that volume's upload is queued, so
    the host's wait for a count never leaves the copy engine idle.  result(ticket) waits for that volume's host
    outputs; they stay valid until `depth` further submissions.  Every step of
    the path runs in libpsn.so's kernels; this class only orders copies and
    launches.
    """

    def __init__(self, psn: PSN, shape, dtype, spacing, iterations: int, relaxation: float, constraint: float,
                 origin=(0.0, 0.0, 0.0), label_set=None, depth: int = 2):
        self.psn, self.shape, self.dtype = psn, tuple(shape), dtype
        self.spacing, self.origin = tuple(spacing), tuple(origin)
        self.T, self.lam, self.d = iterations, relaxation, constraint
        self.labels = psn.labels(label_set)
        self.depth = depth
        self.dev = f"cuda:{psn.device}"
        self.s_h2d, self.s_comp, self.s_d2h = (torch.cuda.Stream(device=self.dev) for _ in range(3))
        self.slots = [dict(labels=torch.empty(self.shape, dtype=dtype, device=self.dev), ws=None, mesh=None,
                           sws=None, out=None, host=None, counts=None, ev_h2d=torch.cuda.Event(),
                           ev_ext=torch.cuda.Event(), ev_comp=torch.cuda.Event(), ev_d2h=torch.cuda.Event(),
                           used=False, computed=False) for _ in range(depth)]
        self._pending = None
        self.n = 0
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def _ensure(self, sl, c):
        """Grow the slot's device mesh / smoothing buffers / pinned outputs to the counted totals."""
        nw = c.halo_lo_points + c.n_points + c.halo_hi_points
        m = sl["mesh"]
        if m is not None and m.points.shape[0] >= nw and m.quads.shape[0] >= c.n_quads and \
                m.stencil_ids.shape[0] >= c.n_stencil and m.stencil_offsets.shape[0] >= c.n_points + 1:
            return
        torch.cuda.synchronize(self.dev)              # rare: old buffers may still be read back
        sl["mesh"] = self.psn.alloc_mesh(nw, c.n_points, c.n_quads, c.n_stencil)
        sl["out"] = torch.empty((max(nw, 1), 3), dtype=torch.float32, device=self.dev)
        sl["host"] = dict(points=torch.empty((max(c.n_points, 1), 3), dtype=torch.float32, pin_memory=True),
                          quads=torch.empty((max(c.n_quads, 1), 4), dtype=torch.int32, pin_memory=True),
                          pairs=torch.empty((max(c.n_quads, 1), 2), dtype=torch.int32, pin_memory=True))
        sl["sws"] = None

    def submit(self, labels_host: torch.Tensor) -> int:
        """Enqueue the upload of one volume, then run the PREVIOUS volume's compute (its PSN_COUNT
        synchronises the host on the compute stream): the copy engine already holds this upload,
        so it never idles while the host waits for a count."""
        if tuple(labels_host.shape) != self.shape or labels_host.dtype != self.dtype:
            raise ValueError("labels_host must match the stream's shape and dtype")
        ticket = self.n
        sl = self.slots[ticket % self.depth]
        with torch.cuda.stream(self.s_h2d):
            if sl["used"]:
                self.s_h2d.wait_event(sl["ev_comp"])         # the slot's previous volume is processed
            sl["labels"].copy_(labels_host, non_blocking=True)
            sl["ev_h2d"].record(self.s_h2d)
        sl["used"] = True
        self.h2d_bytes = labels_host.numel() * labels_host.element_size()
        self.n += 1
        self.flush()
        self._pending = ticket
        return ticket

    def flush(self):
        """Run the compute of the last submitted volume if it is still pending (result() does this)."""
        t = getattr(self, "_pending", None)
        if t is None:
            return
        self._pending = None
        sl = self.slots[t % self.depth]
        vol = self.psn.volume(sl["labels"], spacing=self.spacing, origin=self.origin)
        if sl["ws"] is None:
            sl["ws"] = self.psn.workspace(vol)
        self.s_comp.wait_event(sl["ev_h2d"])
        if sl["computed"]:
            self.s_comp.wait_event(sl["ev_d2h"])               # the slot's previous outputs are read back
        c = self.psn.count(vol, self.labels, sl["ws"], self.s_comp)   # exact totals (one sync)
        self._ensure(sl, c)
        mesh = self.psn.emit(vol, self.labels, sl["ws"], c, mesh=sl["mesh"], stream=self.s_comp)
        sl["ev_ext"].record(self.s_comp)
        if sl["sws"] is None or sl["sws"].numel() < self._sws_bytes(mesh):
            sl["sws"] = self.psn.smooth_workspace(mesh)
        out = self.psn.smooth(vol, mesh, self.T, self.lam, self.d, out=sl["out"], ws=sl["sws"], stream=self.s_comp)
        sl["ev_comp"].record(self.s_comp)
        P, Q = mesh.n_points, mesh.n_quads
        host = sl["host"]
        with torch.cuda.stream(self.s_d2h):
            self.s_d2h.wait_event(sl["ev_ext"])
            host["quads"][:Q].copy_(mesh.quads[:Q], non_blocking=True)
            host["pairs"][:Q].copy_(mesh.pairs[:Q], non_blocking=True)
            self.s_d2h.wait_event(sl["ev_comp"])
            host["points"][:P].copy_(out[:P], non_blocking=True)
            sl["ev_d2h"].record(self.s_d2h)
        sl["counts"] = (P, Q, mesh.n_stencil)
        sl["computed"] = True
        self.d2h_bytes = P * 12 + Q * 24

    def _sws_bytes(self, mesh) -> int:
        n = ctypes.c_size_t()
        self.psn._check(self.psn.L.psn_smooth_workspace(ctypes.byref(mesh.c), ctypes.byref(n)))
        return n.value

    def result(self, ticket: int):
        """(points f32 [P,3], quads i32 [Q,4], pairs i32 [Q,2]) on the host for `ticket`."""
        if not (self.n - self.depth <= ticket < self.n):
            raise ValueError("ticket no longer (or not yet) available")
        if ticket == self._pending:
            self.flush()
        sl = self.slots[ticket % self.depth]
        sl["ev_d2h"].synchronize()
        P, Q, _ = sl["counts"]
        h = sl["host"]
        return h["points"][:P], h["quads"][:Q], h["pairs"][:Q]
