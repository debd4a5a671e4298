"""Plain CPU oracle for the PSN hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product package ``paper_2401_14906_b200`` never imports it, and the two share
no code: this wrapper only marshals numpy arrays into ``liboracle.so``
(``oracle/psn_oracle.c``), whose header documents what each routine computes
and which PAPER.md passage it follows.

Functions
---------
layer_counts(vol, ...)        per-voxel-layer (P, Q, S)
row_trims(vol, ...)           per-grid-row Pass-1 / Pass-2 trims
extract(vol, ...)             points, quads, pairs, CSR, face masks
smooth(mesh, ...)             fp64 Jacobi constrained Laplacian      P:64-69 (Eq. 1)
triangulate(quads, points)    shortest-diagonal split

Parity pins: see tests/test_oracle_pins.py (every function here is pinned
there against closed forms, invariants, brute force or the paper's worked
cases).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "psn_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

BACKGROUND = 0xFFFFFFFF

_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", _LIB_PATH, _SRC])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        vp = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.oracle_layer_counts.restype = ctypes.c_int
        lib.oracle_layer_counts.argtypes = [vp, ctypes.c_int, i64, i64, i64, i64, i64,
                                            vp, i64, ctypes.c_int, i64, i64, vp, vp, vp]
        lib.oracle_row_trims.restype = ctypes.c_int
        lib.oracle_row_trims.argtypes = [vp, ctypes.c_int, i64, i64, i64, i64, i64,
                                         vp, i64, ctypes.c_int, i64, i64, vp, vp, vp, vp]
        lib.oracle_extract.restype = ctypes.c_int
        lib.oracle_extract.argtypes = [vp, ctypes.c_int, i64, i64, i64, i64, i64,
                                       vp, i64, ctypes.c_int, vp, vp,
                                       i64, i64, i64, i64,
                                       vp, vp, vp, vp, vp, vp, vp, vp,
                                       i64, i64, i64, _i64p, _i64p, _i64p]
        lib.oracle_smooth.restype = ctypes.c_int
        lib.oracle_smooth.argtypes = [i64, vp, vp, vp, i64, vp, vp, ctypes.c_int32,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_int, vp]
        lib.oracle_triangulate.restype = ctypes.c_int
        lib.oracle_triangulate.argtypes = [i64, vp, vp, i64, ctypes.c_int, vp]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Volume:
    """Lattice slices [z_lo, z_hi) of a global M x N x O label volume.

    ``labels`` is a numpy array of shape (z_hi - z_lo, N, M) (x fastest),
    dtype uint8 / uint16 / uint32.
    """
    labels: np.ndarray
    dims: tuple  # (M, N, O) global
    z_lo: int = 0
    spacing: tuple = (1.0, 1.0, 1.0)
    origin: tuple = (0.0, 0.0, 0.0)
    label_set: tuple | None = None  # None => all non-zero values (reading Q2)

    @property
    def z_hi(self):
        return self.z_lo + self.labels.shape[0]


def as_volume(labels, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0), label_set=None):
    a = np.ascontiguousarray(labels)
    O, N, M = a.shape
    return Volume(a, (M, N, O), 0, tuple(spacing), tuple(origin), label_set)


def _label_args(vol: Volume):
    if vol.label_set is None:
        return None, 0, 1, None
    L = np.unique(np.asarray(vol.label_set, dtype=np.uint32))
    return L, len(L), 0, L


@dataclass
class Mesh:
    points: np.ndarray      # float32 [P,3]
    anchors: np.ndarray     # float64 [P,3]
    voxel_idx: np.ndarray   # int64 [P,3]
    quads: np.ndarray       # uint32 [Q,4]
    pairs: np.ndarray       # uint32 [Q,2]
    csr_off: np.ndarray     # uint32 [P+1]
    csr_ids: np.ndarray     # uint32 [S]
    face_mask: np.ndarray   # uint8 [P]
    point_base: int = 0
    stencil_base: int = 0

    @property
    def n_points(self):
        return len(self.points)

    @property
    def n_quads(self):
        return len(self.quads)

    @property
    def n_stencil(self):
        return len(self.csr_ids)


def layer_counts(vol: Volume, k0: int = 0, k1: int | None = None):
    """Per voxel layer k in [k0, k1): (P_k, Q_k, S_k) as int64 arrays."""
    lib = _load()
    M, N, O = vol.dims
    if k1 is None:
        k1 = O - 1
    n = max(k1 - k0, 0)
    P = np.zeros(n, np.int64); Q = np.zeros(n, np.int64); S = np.zeros(n, np.int64)
    L, nL, anz, keep = _label_args(vol)
    lab = np.ascontiguousarray(vol.labels)
    rc = lib.oracle_layer_counts(_ptr(lab), lab.dtype.itemsize, M, N, O, vol.z_lo, vol.z_hi,
                                 _ptr(L), nL, anz, k0, k1, _ptr(P), _ptr(Q), _ptr(S))
    if rc != 0:
        raise ValueError(f"oracle_layer_counts: bad arguments (rc={rc})")
    return P, Q, S


def row_trims(vol: Volume, k0: int = 0, k1: int | None = None):
    """Per grid row E_{j,k} (j < N, k in [k0, k1)): (pass1, final) trims, each int64 [k1-k0, N, 2]
    holding [xL, xR): Pass 1 from the x-edges only, final after Pass 2's y/z-edges
    (P:83); empty rows [0, 0)."""
    lib = _load()
    M, N, O = vol.dims
    if k1 is None:
        k1 = O
    n = max(k1 - k0, 0) * N
    a = [np.zeros(n, np.int64) for _ in range(4)]
    L, nL, anz, keep = _label_args(vol)
    lab = np.ascontiguousarray(vol.labels)
    rc = lib.oracle_row_trims(_ptr(lab), lab.dtype.itemsize, M, N, O, vol.z_lo, vol.z_hi,
                              _ptr(L), nL, anz, k0, k1, *(_ptr(x) for x in a))
    if rc != 0:
        raise ValueError(f"oracle_row_trims: bad arguments (rc={rc})")
    shape = (max(k1 - k0, 0), N)
    return np.stack([a[0].reshape(shape), a[1].reshape(shape)], -1), np.stack([a[2].reshape(shape), a[3].reshape(shape)], -1)


def extract(vol: Volume, k0: int = 0, k1: int | None = None, point_base: int = 0,
            stencil_base: int = 0) -> Mesh:
    """Mesh owned by voxel layers [k0, k1) with global ids (see psn_oracle.c)."""
    lib = _load()
    M, N, O = vol.dims
    if k1 is None:
        k1 = O - 1
    L, nL, anz, keep = _label_args(vol)
    lab = np.ascontiguousarray(vol.labels)
    sp = np.asarray(vol.spacing, np.float64); org = np.asarray(vol.origin, np.float64)
    if k1 <= k0:
        return Mesh(np.zeros((0, 3), np.float32), np.zeros((0, 3)), np.zeros((0, 3), np.int64),
                    np.zeros((0, 4), np.uint32), np.zeros((0, 2), np.uint32),
                    np.array([stencil_base], np.uint32), np.zeros(0, np.uint32),
                    np.zeros(0, np.uint8), point_base, stencil_base)
    P, Q, S = layer_counts(vol, k0, k1)
    nP, nQ, nS = int(P.sum()), int(Q.sum()), int(S.sum())
    pts = np.zeros((nP, 3), np.float32); anc = np.zeros((nP, 3), np.float64)
    vidx = np.zeros((nP, 3), np.int64)
    quads = np.zeros((nQ, 4), np.uint32); pairs = np.zeros((nQ, 2), np.uint32)
    off = np.zeros(nP + 1, np.uint32); ids = np.zeros(nS, np.uint32); fm = np.zeros(nP, np.uint8)
    oP, oQ, oS = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    rc = lib.oracle_extract(_ptr(lab), lab.dtype.itemsize, M, N, O, vol.z_lo, vol.z_hi,
                            _ptr(L), nL, anz, _ptr(sp), _ptr(org), k0, k1, point_base, stencil_base,
                            _ptr(pts), _ptr(anc), _ptr(vidx), _ptr(quads), _ptr(pairs),
                            _ptr(off), _ptr(ids), _ptr(fm), nP, nQ, nS,
                            ctypes.byref(oP), ctypes.byref(oQ), ctypes.byref(oS))
    if rc != 0:
        raise RuntimeError(f"oracle_extract failed rc={rc}")
    assert (oP.value, oQ.value, oS.value) == (nP, nQ, nS)
    return Mesh(pts, anc, vidx, quads, pairs, off, ids, fm, point_base, stencil_base)


BOX, SPHERE = 0, 1


def smooth(mesh: Mesh, spacing, iterations: int, relaxation: float, constraint: float,
           frozen: np.ndarray | None = None, shape: int = BOX) -> np.ndarray:
    """fp64 Jacobi constrained Laplacian smoothing (Eq. 1); returns float64 [P,3] world coords.
    shape BOX: |p - anchor|_a <= d*s_a per axis; SPHERE: |p - anchor| <= d*min(s)."""
    lib = _load()
    nP = mesh.n_points
    out = np.zeros((nP, 3), np.float64)
    sp = np.asarray(spacing, np.float64)
    fz = None if frozen is None else np.ascontiguousarray(frozen, np.uint8)
    rc = lib.oracle_smooth(nP, _ptr(np.ascontiguousarray(mesh.anchors)), _ptr(mesh.csr_off),
                           _ptr(mesh.csr_ids), mesh.point_base, _ptr(fz), _ptr(sp),
                           int(iterations), float(relaxation), float(constraint), int(shape), _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle_smooth: bad arguments rc={rc}")
    return out


FIXED_02, SHORTEST, MIN_AREA, MOST_COPLANAR = 0, 1, 2, 3


def triangulate(quads: np.ndarray, points: np.ndarray, id_base: int = 0, strategy: int = SHORTEST):
    """Two triangles per quad: 0 = fixed 0-2, 1 = shorter diagonal, 2 = minimum area,
    3 = most co-planar; ties -> 0-2."""
    lib = _load()
    q = np.ascontiguousarray(quads, np.uint32)
    p = np.ascontiguousarray(points, np.float32)
    tris = np.zeros((len(q) * 2, 3), np.uint32)
    rc = lib.oracle_triangulate(len(q), _ptr(q), _ptr(p), id_base, strategy, _ptr(tris))
    if rc != 0:
        raise ValueError("oracle_triangulate: bad strategy")
    return tris
