"""Independent formulations used to PIN the oracle (tests only).

None of this shares code with oracle/psn_oracle.c: it restates what the paper
fixes in a different form (vectorised corner / face counting, the textbook
cuberille surface, closed forms), so that a dropped term, a wrong sign or
index, or a transposed operand in the oracle fails a test.
"""
from __future__ import annotations

import numpy as np

B = 0xFFFFFFFF


def classes(labels: np.ndarray, label_set=None) -> np.ndarray:
    """cls(v) = v if v in L else B, as int64 (reading Q1)."""
    a = labels.astype(np.int64)
    if label_set is None:
        inl = a != 0
    else:
        inl = np.isin(a, np.asarray(list(label_set), np.int64))
    return np.where(inl, a, np.int64(B))


def corner_point_mask(C: np.ndarray) -> np.ndarray:
    """Voxel (k,j,i) has a point iff its 8 corner classes are not all equal
    (equivalent to 'any of 12 edges intersected').  Shape (O-1,N-1,M-1)."""
    c0 = C[:-1, :-1, :-1]
    diff = np.zeros(c0.shape, bool)
    for dk in (0, 1):
        for dj in (0, 1):
            for di in (0, 1):
                diff |= C[dk:C.shape[0] - 1 + dk, dj:C.shape[1] - 1 + dj, di:C.shape[2] - 1 + di] != c0
    return diff


def count_identities(C: np.ndarray):
    """(P, Q, S) from counting identities (SURVEY 8(c) 'What pins each part'):
    P = #voxels with non-uniform corners; Q = #lattice edges with I=1 whose four
    sharing voxels exist; S = 2 * #faces shared by two voxels whose 4 corners
    are not all equal."""
    O, N, M = C.shape
    P = int(corner_point_mask(C).sum())
    Q = 0
    # x-edges (i,i+1) at (j,k): sharing voxels j-1..j, k-1..k -> 1<=j<=N-2, 1<=k<=O-2
    ex = C[:, :, 1:] != C[:, :, :-1]
    Q += int(ex[1:O - 1, 1:N - 1, :].sum())
    ey = C[:, 1:, :] != C[:, :-1, :]
    Q += int(ey[1:O - 1, :, 1:M - 1].sum())
    ez = C[1:, :, :] != C[:-1, :, :]
    Q += int(ez[:, 1:N - 1, 1:M - 1].sum())
    S = 0
    # a face perpendicular to x at lattice plane i (1<=i<=M-2) between voxels i-1 and i,
    # spanning lattice points (j..j+1, k..k+1): non-uniform corners
    def nonuni(f):  # f: list of 4 arrays
        return (f[1] != f[0]) | (f[2] != f[0]) | (f[3] != f[0])
    fx = nonuni([C[:-1, :-1, :], C[:-1, 1:, :], C[1:, :-1, :], C[1:, 1:, :]])  # (O-1,N-1,M)
    S += 2 * int(fx[:, :, 1:M - 1].sum())
    fy = nonuni([C[:-1, :, :-1], C[:-1, :, 1:], C[1:, :, :-1], C[1:, :, 1:]])  # (O-1,N,M-1)
    S += 2 * int(fy[:, 1:N - 1, :].sum())
    fz = nonuni([C[:, :-1, :-1], C[:, :-1, 1:], C[:, 1:, :-1], C[:, 1:, 1:]])  # (O,N-1,M-1)
    S += 2 * int(fz[1:O - 1, :, :].sum())
    return P, Q, S


def cuberille_faces(C: np.ndarray):
    """Textbook dual surface: for every lattice edge whose endpoints differ in
    class and whose four sharing voxels exist, the unit square dual to it.
    Returns {frozenset of 4 voxel (i,j,k)}: (axis, origin lattice point, far lattice point)."""
    O, N, M = C.shape
    out = {}
    for axis, (di, dj, dk) in enumerate(((1, 0, 0), (0, 1, 0), (0, 0, 1))):
        kk, jj, ii = np.nonzero(C[dk:, dj:, di:] != C[:O - dk, :N - dj, :M - di])
        for i, j, k in zip(ii.tolist(), jj.tolist(), kk.tolist()):
            # the 4 voxels sharing the edge: offsets -1/0 in the two other axes
            others = [a for a in range(3) if a != axis]
            vox = []
            ok = True
            for s0 in (-1, 0):
                for s1 in (-1, 0):
                    v = [i, j, k]
                    v[others[0]] += s0
                    v[others[1]] += s1
                    if not (0 <= v[0] < M - 1 and 0 <= v[1] < N - 1 and 0 <= v[2] < O - 1):
                        ok = False
                    vox.append(tuple(v))
            if ok:
                far = (i + di, j + dj, k + dk)
                out[frozenset(vox)] = (axis, (i, j, k), far)
    return out


def quad_normal(centres: np.ndarray) -> np.ndarray:
    """(q2-q0) x (q3-q1) for a [4,3] array of vertex positions."""
    return np.cross(centres[2] - centres[0], centres[3] - centres[1])


def euler_characteristic(quads: np.ndarray) -> int:
    """V - E + F over the vertices / undirected edges / faces used by quads."""
    if len(quads) == 0:
        return 0
    verts = set(np.unique(quads).tolist())
    edges = set()
    for q in quads.tolist():
        for a in range(4):
            u, v = q[a], q[(a + 1) % 4]
            edges.add((min(u, v), max(u, v)))
    return len(verts) - len(edges) + len(quads)


def edge_multiplicity(quads: np.ndarray):
    m = {}
    for q in quads.tolist():
        for a in range(4):
            u, v = q[a], q[(a + 1) % 4]
            e = (min(u, v), max(u, v))
            m[e] = m.get(e, 0) + 1
    return m


def directed_edges(quads: np.ndarray):
    m = {}
    for q in quads.tolist():
        for a in range(4):
            e = (q[a], q[(a + 1) % 4])
            m[e] = m.get(e, 0) + 1
    return m
