"""Pins for the oracle (CPU only, no GPU).

Each test checks oracle/ against something other than itself: the worked
cases the paper/spec print (tests/golden/worked_cases.txt), counting
identities and the textbook cuberille surface written independently in
tests/indep.py, closed forms (digital balls, the dual-cube smoothing decay,
iid expectations), invariants, and brute force over all 2x2x2 volumes.
See DESIGN.md section 4 for the list and what each pin would catch.
"""
import itertools
import math

import numpy as np
import pytest

import golden_cases
import indep
import oracle

GOLD = golden_cases.load()


def extract(a, **kw):
    return oracle.extract(oracle.as_volume(a, **kw))


# --------------------------------------------------------------------------- worked cases
def test_single_point_golden():
    case = GOLD["single_point_3"]
    a = golden_cases.volume(case)
    m = extract(a)
    P, Q, S = (int(x) for x in case["expect_counts"].split())
    assert (m.n_points, m.n_quads, m.n_stencil) == (P, Q, S)
    assert np.all(np.diff(m.csr_off) == int(case["expect_degree"]))
    assert indep.euler_characteristic(m.quads) == int(case["expect_euler"])
    # the 8 points are the 8 voxel centres, in row-major order
    exp = np.array([[i + 0.5, j + 0.5, k + 0.5] for k in (0, 1) for j in (0, 1) for i in (0, 1)], np.float32)
    np.testing.assert_array_equal(m.points, exp)
    # every quad edge shared by exactly two quads (closed dual cube)
    assert set(indep.edge_multiplicity(m.quads).values()) == {2}


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.uint32])
def test_single_point_golden_arrays(dtype):
    """The 3^3 worked case written out array by array (tests/golden/worked_cases.txt,
    single_point_3_arrays): quads IN ORDER with their pairs, CSR offsets and ids, face masks.
    Pins the output ORDER (reading Q4: voxel-major, then x<y<z) that the counting pins cannot see."""
    case = GOLD["single_point_3_arrays"]
    a = golden_cases.volume(case, dtype)
    m = extract(a)
    quads = np.array([[int(x) for x in q.split("|")[0].split()] for q in case["mquads"]], np.uint32)
    pairs = np.array([[int(x) for x in q.split("|")[1].split()] for q in case["mquads"]], np.uint32)
    np.testing.assert_array_equal(m.quads, quads)
    np.testing.assert_array_equal(m.pairs, pairs)
    np.testing.assert_array_equal(m.csr_off, np.array(case["csr_off"].split(), np.uint32))
    np.testing.assert_array_equal(m.csr_ids, np.array(case["csr_ids"].split(), np.uint32))
    np.testing.assert_array_equal(m.face_mask, np.array(case["face_mask"].split(), np.uint8))
    np.testing.assert_array_equal(m.voxel_idx, np.array([[i, j, k] for k in (0, 1) for j in (0, 1) for i in (0, 1)]))


def test_pass1_rows_golden():
    """S:218-220 Pass-1 row examples: the x-intersections and the trim [xL, xR) of a
    row.  Each row is embedded as grid row (j=1, k=1) of an M x 3 x 3 volume whose other rows are
    background: the oracle's Pass-1 trim of that row is the printed one, and its x-quads (owned by
    voxels (i,1,1)) sit exactly at the printed x-intersections."""
    for spec in GOLD["pass1_rows"]["rows"]:
        vals, _, rest = spec.partition("->")
        xs, _, trim = rest.partition("|")
        row = [int(x) for x in vals.split()]
        xint = [int(x) for x in xs.split()]
        xl, xr = (int(x) for x in trim.split())
        M = len(row)
        a = np.zeros((3, 3, M), np.uint16)
        a[1, 1, :] = row
        vol = oracle.as_volume(a)
        p1, fin = oracle.row_trims(vol)
        assert tuple(p1[1, 1]) == (xl, xr), (spec, p1[1, 1])
        m = oracle.extract(vol)
        vi = m.voxel_idx
        xq = sorted(int(vi[q[2], 0]) for q in m.quads.tolist()
                    if len({int(vi[v, 0]) for v in q}) == 1 and tuple(vi[q[2], 1:]) == (1, 1))
        assert xq == xint, (spec, xq)
        # rows holding no intersection at all have empty trims [0, 0)
        assert tuple(p1[0, 0]) == (0, 0) and tuple(fin[0, 0]) == (0, 0)


def _indep_trims(C):
    """Pass-1 / Pass-2 trims of every grid row written with numpy edge planes (independent of
    the oracle's loops): [first, last + 1) of the X (resp. X|Y|Z) intersections, [0, 0) if none."""
    O, N, M = C.shape
    X = np.zeros(C.shape, bool); Y = np.zeros(C.shape, bool); Z = np.zeros(C.shape, bool)
    X[:, :, :-1] = C[:, :, 1:] != C[:, :, :-1]
    Y[:, :-1, :] = C[:, 1:, :] != C[:, :-1, :]
    Z[:-1, :, :] = C[1:, :, :] != C[:-1, :, :]

    def tr(E):
        any_ = E.any(-1)
        first = np.argmax(E, -1)
        last = M - 1 - np.argmax(E[..., ::-1], -1)
        return np.stack([np.where(any_, first, 0), np.where(any_, last + 1, 0)], -1)
    return tr(X), tr(X | Y | Z)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.uint32])
def test_row_trims_tight_and_sound(dtype):
    """Trims: equal to the tightest intervals of the numpy edge planes, Pass-1
    inside Pass-2, and SOUND: every point-producing voxel of voxel row (j,k) lies in
    [max(0, minL-1), min(maxR, M-1)) over the four grid rows (j..j+1, k..k+1)."""
    rng = np.random.default_rng(42)
    for t in range(60):
        a = _random_volume(rng, max_dim=11, dtype=dtype)
        if dtype == np.uint32:
            a = (a.astype(np.uint64) * 0x10001 + 0x7F000000).astype(np.uint32) * (a != 0)
        nz = [v for v in np.unique(a).tolist() if v != 0]
        ls = None if t % 2 == 0 else (nz[:2] or None)
        vol = oracle.as_volume(a, label_set=ls)
        p1, fin = oracle.row_trims(vol)
        e1, ef = _indep_trims(indep.classes(a, ls))
        np.testing.assert_array_equal(p1, e1)
        np.testing.assert_array_equal(fin, ef)
        nonempty = p1[..., 1] > p1[..., 0]
        assert np.all(fin[nonempty, 0] <= p1[nonempty, 0]) and np.all(fin[nonempty, 1] >= p1[nonempty, 1])
        m = oracle.extract(vol)
        O, N, M = a.shape
        for i, j, k in m.voxel_idx.tolist():
            rows = [fin[kk, jj] for kk in (k, k + 1) for jj in (j, j + 1) if fin[kk, jj, 1] > fin[kk, jj, 0]]
            assert rows, "a point in a voxel row whose four grid rows have no intersection"
            lo = max(0, min(r[0] for r in rows) - 1)
            hi = min(max(r[1] for r in rows), M - 1)
            assert lo <= i < hi


def _u32_volume(rng, max_dim=10):
    """u32 labels that agree in their low 16 (and low 8) bits but differ above: a reader that
    truncated to u16 / u8 would merge them."""
    a = _random_volume(rng, max_dim=max_dim, nlab=4).astype(np.uint64)
    hi = np.array([0, 0x00010000, 0x7FFF0000, 0xFFFE0000], np.uint64)
    return np.where(a == 0, 0, (a & 1) + 0x5 + hi[a]).astype(np.uint32)


def test_u32_counting_identities_and_cuberille():
    """The u32 read path (psn_oracle.c o_raw elem_bytes 4): counting identities and the textbook
    cuberille surface on u32 volumes whose labels collide in their low bits, incl. label subsets
    of large values and the largest non-sentinel value 0xFFFFFFFE."""
    rng = np.random.default_rng(2024)
    for t in range(40):
        a = _u32_volume(rng)
        if t % 4 == 3:
            a[a.shape[0] // 2, :, : a.shape[2] // 2] = 0xFFFFFFFE
        vals = [v for v in np.unique(a).tolist() if v != 0]
        ls = None if t % 2 == 0 or not vals else vals[: max(1, len(vals) // 2)]
        P, Q, S = oracle.layer_counts(oracle.as_volume(a, label_set=ls))
        C = indep.classes(a, ls)
        assert (int(P.sum()), int(Q.sum()), int(S.sum())) == indep.count_identities(C)
        if t % 2 == 0:
            m = _check_against_cuberille(a, label_set=ls)
            # low-bit collisions really occur and really intersect
            assert set(m.pairs.ravel().tolist()) <= set(np.unique(C).tolist())
    # two labels equal in the low 16 bits: the interface between them is a surface
    a = np.zeros((4, 4, 5), np.uint32)
    a[1:3, 1:3, 1:3] = 0x00010001
    a[1:3, 1:3, 3] = 0x00000001
    m = extract(a)
    assert [tuple(p) for p in m.pairs.tolist()].count((0x00010001, 0x00000001)) == 4


@pytest.mark.parametrize("n", [3, 5, 6])
def test_single_point_any_size(n):
    a = np.zeros((n, n, n), np.uint8)
    c = n // 2
    a[c, c, c] = 9
    m = extract(a)
    assert (m.n_points, m.n_quads, m.n_stencil) == (8, 6, 24)
    assert indep.euler_characteristic(m.quads) == 2


def test_two_adjacent_labels():
    case = GOLD["two_adjacent_labels_4"]
    a = golden_cases.volume(case)
    m = extract(a)
    l0, l1, cnt = (int(x) for x in case["expect_pair_count"].split())
    pairs = [tuple(p) for p in m.pairs.tolist()]
    assert pairs.count((l0, l1)) == cnt
    assert (m.n_points, m.n_quads, m.n_stencil) == indep.count_identities(indep.classes(a))
    # each label's submesh is a closed dual cube (6 quads), sharing the (1,2) quad
    for lab in (l0, l1):
        sub = m.quads[(m.pairs == lab).any(1)]
        assert len(sub) == 6
        assert set(indep.edge_multiplicity(sub).values()) == {2}


@pytest.mark.parametrize("name", ["all_background_8", "uniform_label_8"])
def test_degenerate(name):
    case = GOLD[name]
    a = golden_cases.volume(case)
    m = extract(a)
    assert (m.n_points, m.n_quads, m.n_stencil) == tuple(int(x) for x in case["expect_counts"].split())
    assert m.csr_off.tolist() == [0]


def test_unselected_label_is_background():
    """Reading Q1: an unselected label next to background is background (no edge)."""
    a = np.zeros((5, 5, 5), np.uint16)
    a[2, 2, 2] = 1
    a[2, 2, 3] = 7  # adjacent, but not in L
    m = oracle.extract(oracle.as_volume(a, label_set=[1]))
    assert (m.n_points, m.n_quads) == (8, 6)
    assert set(m.pairs.ravel().tolist()) == {1, oracle.BACKGROUND}
    # with 7 selected, a shared (1,7) quad appears
    m2 = oracle.extract(oracle.as_volume(a, label_set=[1, 7]))
    assert [tuple(p) for p in m2.pairs.tolist()].count((1, 7)) == 1


def test_stacked_slabs_yz_only():
    """P:124 pathological case: two uniform slabs stacked in y -> only y-edges
    intersect (empty x-trims).  Closed forms for an M x N x O volume."""
    for M, N, O in [(6, 4, 5), (9, 4, 7), (3, 4, 3)]:
        a = np.ones((O, N, M), np.uint16)
        a[:, 2:, :] = 2
        m = extract(a)
        P = (M - 1) * (O - 1)
        Q = (M - 2) * (O - 2)
        S = 2 * ((M - 2) * (O - 1) + (M - 1) * (O - 2))
        assert (m.n_points, m.n_quads, m.n_stencil) == (P, Q, S)
        assert np.all(m.pairs == np.array([1, 2], np.uint32))


# --------------------------------------------------------------------------- counting identities
def _random_volume(rng, max_dim=12, dtype=np.uint16, nlab=5):
    M, N, O = (int(rng.integers(2, max_dim + 1)) for _ in range(3))
    a = rng.integers(0, nlab, size=(O, N, M)).astype(dtype)
    # blobs: sometimes smooth regions instead of noise
    if rng.random() < 0.5:
        z, y, x = np.meshgrid(np.arange(O), np.arange(N), np.arange(M), indexing="ij")
        a = ((x // rng.integers(1, 4) + y // rng.integers(1, 4) + z // rng.integers(1, 4)) % nlab).astype(dtype)
    return a


def test_counting_identities_random():
    rng = np.random.default_rng(1234)
    for t in range(150):
        a = _random_volume(rng)
        ls = None
        if t % 3 == 1:
            ls = sorted(set(rng.integers(0, 5, size=rng.integers(1, 4)).tolist()))
        P, Q, S = oracle.layer_counts(oracle.as_volume(a, label_set=ls))
        assert (int(P.sum()), int(Q.sum()), int(S.sum())) == indep.count_identities(indep.classes(a, ls))


def test_layer_counts_match_extract_and_corner_mask():
    rng = np.random.default_rng(7)
    for _ in range(40):
        a = _random_volume(rng, max_dim=10)
        C = indep.classes(a)
        m = extract(a)
        pm = indep.corner_point_mask(C)
        # ids are assigned in row-major voxel order: voxel_idx is exactly the nonzero list of pm
        kk, jj, ii = np.nonzero(pm)
        np.testing.assert_array_equal(m.voxel_idx, np.stack([ii, jj, kk], 1))
        P, Q, S = oracle.layer_counts(oracle.as_volume(a))
        assert (P.sum(), Q.sum(), S.sum()) == (m.n_points, m.n_quads, m.n_stencil)


# --------------------------------------------------------------------------- cuberille / orientation
def _check_against_cuberille(a, label_set=None, spacing=(1.0, 1.0, 1.0)):
    C = indep.classes(a, label_set)
    m = oracle.extract(oracle.as_volume(a, spacing=spacing, label_set=label_set))
    faces = indep.cuberille_faces(C)
    vidx = m.voxel_idx
    got = {}
    for q, pr in zip(m.quads.tolist(), m.pairs.tolist()):
        vox = frozenset(tuple(vidx[v].tolist()) for v in q)
        assert len(vox) == 4
        assert vox not in got, "duplicate quad"
        got[vox] = (q, pr)
    assert set(got) == set(faces)
    for vox, (axis, org, far) in faces.items():
        q, pr = got[vox]
        assert pr == [int(C[org[2], org[1], org[0]]), int(C[far[2], far[1], far[0]])]
        n = indep.quad_normal(m.anchors[q])
        # normal along +axis (from pair[0]'s region into pair[1]'s), reading Q6
        assert n[axis] > 0 and abs(n[(axis + 1) % 3]) < 1e-9 and abs(n[(axis + 2) % 3]) < 1e-9
        assert q[0] == min(q)
    return m


def test_cuberille_binary_random():
    rng = np.random.default_rng(99)
    for _ in range(60):
        M, N, O = (int(rng.integers(2, 9)) for _ in range(3))
        a = (rng.random((O, N, M)) < rng.uniform(0.1, 0.7)).astype(np.uint8)
        _check_against_cuberille(a)


def test_cuberille_multilabel_random():
    rng = np.random.default_rng(5)
    for _ in range(40):
        a = _random_volume(rng, max_dim=8, nlab=4)
        _check_against_cuberille(a, spacing=(0.8, 1.1, 1.5))


# --------------------------------------------------------------------------- balls: closed manifolds
def _ball(n, c, r):
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    return (((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2) <= r * r).astype(np.uint8)


def test_digital_balls_closed_manifold():
    rng = np.random.default_rng(3)
    done = 0
    while done < 40:
        r = rng.uniform(0.5, 5.0)
        n = int(2 * math.ceil(r) + 5)
        c = rng.uniform(math.ceil(r) + 1.5, n - math.ceil(r) - 2.5, size=3)
        a = _ball(n, c, r)
        if a.sum() == 0:
            continue
        m = extract(a)
        assert set(indep.edge_multiplicity(m.quads).values()) == {2}
        assert indep.euler_characteristic(m.quads) == 2
        assert m.n_points == m.n_quads + 2
        assert m.n_stencil == 4 * m.n_quads
        # every vertex link is a single cycle
        nbr = {}
        for q in m.quads.tolist():
            for t in range(4):
                nbr.setdefault(q[t], []).append((q[(t - 1) % 4], q[(t + 1) % 4]))
        for v, es in nbr.items():
            adj = {}
            for u, w in es:
                adj.setdefault(u, []).append(w)
                adj.setdefault(w, []).append(u)
            assert all(len(x) == 2 for x in adj.values())
            seen, stack = set(), [next(iter(adj))]
            while stack:
                u = stack.pop()
                if u in seen:
                    continue
                seen.add(u)
                stack.extend(adj[u])
            assert len(seen) == len(adj)
        done += 1


def test_multilabel_oriented_closedness():
    """Per label l >= 1 voxel from every face: orient each l-quad out of l; the
    directed edge chain has zero boundary and undirected multiplicity is even
    (2 or 4; SPEC S:279 'exactly two' holds only for balls -- reading Q22)."""
    rng = np.random.default_rng(11)
    for _ in range(40):
        n = int(rng.integers(6, 11))
        a = np.zeros((n, n, n), np.uint16)
        a[2:-2, 2:-2, 2:-2] = rng.integers(0, 4, size=(n - 4, n - 4, n - 4))
        m = extract(a)
        for lab in set(np.unique(a).tolist()) - {0}:
            sel = (m.pairs == lab).any(1)
            q = m.quads[sel].copy()
            flip = m.pairs[sel][:, 1] == lab
            q[flip] = q[flip][:, ::-1]
            d = indep.directed_edges(q)
            for (u, v), c in d.items():
                assert d.get((v, u), 0) == c
            assert all(c % 2 == 0 for c in indep.edge_multiplicity(q).values())


def test_stencil_structure():
    rng = np.random.default_rng(17)
    for _ in range(40):
        a = _random_volume(rng, max_dim=10)
        m = extract(a)
        off, ids = m.csr_off.astype(np.int64), m.csr_ids.astype(np.int64)
        assert off[0] == 0 and off[-1] == len(ids)
        deg = np.diff(off)
        assert deg.max(initial=0) <= 6
        # popcount(face mask) == degree
        pc = np.array([bin(x).count("1") for x in m.face_mask.tolist()], np.int64)
        np.testing.assert_array_equal(pc, deg)
        edges = set()
        for p in range(m.n_points):
            row = ids[off[p]:off[p + 1]]
            assert np.all(np.diff(row) > 0)  # ascending ids (face order)
            for qn in row.tolist():
                edges.add((p, qn))
                d = np.abs(m.voxel_idx[p] - m.voxel_idx[qn])
                assert d.sum() == 1  # face-adjacent voxels
        assert all((b, a2) in edges for a2, b in edges)  # symmetric
        # quad sides are stencil pairs
        for q in m.quads.tolist():
            for t in range(4):
                assert (q[t], q[(t + 1) % 4]) in edges


# --------------------------------------------------------------------------- iid expectation
def test_iid_expectations():
    """c5a-like iid {0,1,2,3}, L = {1,2,3}: analytic expectations."""
    rng = np.random.default_rng(2024)
    n = 48
    a = rng.integers(0, 4, size=(n, n, n)).astype(np.uint8)
    P, Q, S = (int(x.sum()) for x in oracle.layer_counts(oracle.as_volume(a)))
    v = (n - 1) ** 3
    EP = v * (1 - 4 / 4 ** 8)
    EQ = 0.75 * 3 * (n - 1) * (n - 2) ** 2
    ES = 2 * 3 * (n - 2) * (n - 1) ** 2 * (63 / 64)
    assert abs(P - EP) < 8 * math.sqrt(v * (4 / 4 ** 8)) + 1
    assert abs(Q - EQ) < 8 * math.sqrt(3 * (n - 1) * (n - 2) ** 2 * 0.1875)
    assert abs(S - ES) < 8 * 2 * math.sqrt(3 * (n - 2) * (n - 1) ** 2 * (63 / 64) * (1 / 64))


# --------------------------------------------------------------------------- brute force 2x2x2
@pytest.mark.parametrize("nval", [2, 3])
def test_bruteforce_2x2x2(nval):
    for vals in itertools.product(range(nval), repeat=8):
        a = np.array(vals, np.uint8).reshape(2, 2, 2)
        m = extract(a)
        C = indep.classes(a)
        allsame = len(set(C.ravel().tolist())) == 1
        assert m.n_points == (0 if allsame else 1)
        # a single voxel: no interior edges -> no quads; no neighbour voxels -> no stencil
        assert m.n_quads == 0 and m.n_stencil == 0
        if m.n_points:
            # face mask: face f set iff that face's 4 corners are not all equal
            f = m.face_mask[0]
            faces = {0: C[0, :, :], 1: C[:, 0, :], 2: C[:, :, 0], 3: C[:, :, 1], 4: C[:, 1, :], 5: C[1, :, :]}
            # stencil needs an existing neighbour; none here, so the mask is 0 (C-5)
            assert f == 0
            assert any(len(set(v.ravel().tolist())) > 1 for v in faces.values())


def test_bruteforce_pairs_of_voxels():
    """All binary 3x2x2 and 2x3x2 and 2x2x3 volumes (two voxels sharing one face):
    stencil entries exist iff the shared face's 4 corners are not uniform."""
    for shape, axis in [((2, 2, 3), 2), ((2, 3, 2), 1), ((3, 2, 2), 0)]:
        for vals in itertools.product(range(2), repeat=12):
            a = np.array(vals, np.uint8).reshape(shape)
            C = indep.classes(a)
            P, Q, S = indep.count_identities(C)
            mm = extract(a)
            assert (mm.n_points, mm.n_quads, mm.n_stencil) == (P, Q, S)


# --------------------------------------------------------------------------- smoothing pins
def test_smoothing_zero_iterations_or_lambda():
    rng = np.random.default_rng(0)
    a = _random_volume(rng, max_dim=9)
    m = extract(a, spacing=(0.8, 0.8, 1.5), origin=(1.0, -2.0, 3.0))
    np.testing.assert_array_equal(oracle.smooth(m, (0.8, 0.8, 1.5), 0, 0.5, 0.5), m.anchors)
    np.testing.assert_array_equal(oracle.smooth(m, (0.8, 0.8, 1.5), 7, 0.0, 0.5), m.anchors)


@pytest.mark.parametrize("lam", [0.25, 0.5, 1.0])
@pytest.mark.parametrize("T", [1, 10, 25])
def test_smoothing_dual_cube_closed_form(lam, T):
    """Single labelled point: each point at centre +- h_t per axis with
    h_t = 0.5 (1 - 2 lambda/3)^t (derived from Eq. 1; the clamp never binds)."""
    a = np.zeros((3, 3, 3), np.uint8)
    a[1, 1, 1] = 1
    sp = (1.0, 2.0, 0.5)
    m = extract(a, spacing=sp)
    out = oracle.smooth(m, sp, T, lam, 0.5)
    h = 0.5 * (1 - 2 * lam / 3) ** T
    centre = np.array([1.0, 1.0, 1.0]) * sp
    exp = centre + np.sign(m.anchors - centre) * h * np.array(sp)
    assert np.max(np.abs(out - exp)) < 1e-13


def test_smoothing_chain_eq1():
    case = GOLD["smooth_chain"]
    xs = [float(x) for x in case["chain_x"].split()]
    m = oracle.Mesh(points=np.zeros((3, 3), np.float32),
                    anchors=np.array([[x, 0.0, 0.0] for x in xs]),
                    voxel_idx=np.zeros((3, 3), np.int64), quads=np.zeros((0, 4), np.uint32),
                    pairs=np.zeros((0, 2), np.uint32), csr_off=np.array([0, 1, 3, 4], np.uint32),
                    csr_ids=np.array([1, 0, 2, 1], np.uint32), face_mask=np.zeros(3, np.uint8))
    out = oracle.smooth(m, (1.0, 1.0, 1.0), 1, float(case["lambda"]), 100.0)
    assert out[1, 0] == float(case["expect_middle"])


def test_smoothing_box_constraint():
    """only the axis that exceeds the half-width is clamped."""
    m = oracle.Mesh(points=np.zeros((2, 3), np.float32),
                    anchors=np.array([[0.0, 0.0, 0.0], [0.1, 3.0, 0.05]]),
                    voxel_idx=np.zeros((2, 3), np.int64), quads=np.zeros((0, 4), np.uint32),
                    pairs=np.zeros((0, 2), np.uint32), csr_off=np.array([0, 1, 2], np.uint32),
                    csr_ids=np.array([1, 0], np.uint32), face_mask=np.zeros(2, np.uint8))
    out = oracle.smooth(m, (1.0, 1.0, 1.0), 1, 1.0, 0.5)
    # point 0: candidate (0.1, 3.0, 0.05) -> y clamped to +0.5 only
    np.testing.assert_array_equal(out[0], [0.1, 0.5, 0.05])


def test_smoothing_containment_and_clamp_binding():
    rng = np.random.default_rng(8)
    n = 20
    a = rng.integers(0, 4, size=(n, n, n)).astype(np.uint8)
    sp = (0.8, 1.0, 1.5)
    m = extract(a, spacing=sp)
    d = 0.5
    out = oracle.smooth(m, sp, 10, 0.5, d)
    dev = np.abs(out - m.anchors) / np.array(sp)
    assert dev.max() <= d * (1 + 1e-12)
    assert (np.isclose(dev, d)).mean() > 0.005  # the clamp binds on iid data


def test_smoothing_symmetry_ball():
    """A ball centred on a lattice point keeps its octahedral symmetry."""
    for c in (7.0, 7.5):
        a = _ball(16, (c, c, c), 4.3)
        m = extract(a)
        out = oracle.smooth(m, (1, 1, 1), 10, 0.5, 0.5)
        centre = c + 0.0  # lattice/half-lattice centre in world units (voxel centre offset included)
        lookup = {tuple(v): i for i, v in enumerate(m.voxel_idx.tolist())}
        for i, v in enumerate(m.voxel_idx.tolist()):
            # reflection x -> 2c - x maps voxel centre i+0.5 to 2c - i - 0.5 = voxel (2c-1-i)
            w = (int(2 * centre - 1 - v[0]), v[1], v[2])
            j = lookup[w]
            assert abs(out[j, 0] - (2 * centre - out[i, 0])) < 1e-12
            assert abs(out[j, 1] - out[i, 1]) < 1e-12
            # axis permutation (x <-> y)
            j2 = lookup[(v[1], v[0], v[2])]
            assert abs(out[j2, 0] - out[i, 1]) < 1e-12 and abs(out[j2, 1] - out[i, 0]) < 1e-12


def test_smoothing_anisotropy_equivariance():
    """Box-mode Jacobi is per-axis affine-equivariant (reading Q11)."""
    rng = np.random.default_rng(4)
    a = _random_volume(rng, max_dim=10, nlab=3)
    sp, org = (0.8, 0.8, 1.5), (10.0, -3.0, 2.5)
    m1 = extract(a)
    m2 = extract(a, spacing=sp, origin=org)
    o1 = oracle.smooth(m1, (1, 1, 1), 12, 0.5, 0.5)
    o2 = oracle.smooth(m2, sp, 12, 0.5, 0.5)
    np.testing.assert_allclose(o2, np.array(org) + o1 * np.array(sp), rtol=0, atol=1e-12)


def test_smoothing_planar_interface_fixed():
    """Jacobi locality: a planar y-interface keeps its normal coordinate exactly."""
    a = np.ones((6, 5, 7), np.uint16)
    a[:, 2:, :] = 2
    m = extract(a)
    out = oracle.smooth(m, (1, 1, 1), 25, 0.5, 0.5)
    assert np.all(out[:, 1] == m.anchors[:, 1])


@pytest.mark.parametrize("lam", [0.5, 1.0])
@pytest.mark.parametrize("sp", [(1.0, 1.0, 1.0), (0.8, 0.8, 1.5)])
def test_smoothing_sphere_dual_cube_closed_form(lam, sp):
    """Sphere constraint ("a constraint sphere centered at the voxel center point"; reading
    Q26: radius r = d*min(s)).  For the dual cube every point moves along its voxel diagonal, whose
    world direction is s (up to signs), by (0.5 - h_t)|s| with h_t = 0.5 (1 - 2 lambda/3)^t; the
    sphere binds once that exceeds r and then holds the point at distance r on the same diagonal
    (the next update points the same way).  So, per axis, offset = max(h_t, 0.5 - r/|s|) in
    voxel units for every t (derived by hand from Eq. 1)."""
    a = np.zeros((3, 3, 3), np.uint8)
    a[1, 1, 1] = 1
    m = extract(a, spacing=sp)
    d = 0.5
    r = d * min(sp)
    s = np.array(sp)
    centre = np.array([1.0, 1.0, 1.0]) * s
    bound = 0.5 - r / np.linalg.norm(s)
    for T in (1, 2, 3, 4, 10, 25):
        out = oracle.smooth(m, sp, T, lam, d, shape=oracle.SPHERE)
        h = max(0.5 * (1 - 2 * lam / 3) ** T, bound)
        exp = centre + np.sign(m.anchors - centre) * h * s
        assert np.max(np.abs(out - exp)) < 1e-12, (T, np.max(np.abs(out - exp)))
    # with lambda = 0.5 the sphere is free for t <= 2 and binds from t = 3 on (unit spacing)
    if sp == (1.0, 1.0, 1.0) and lam == 0.5:
        assert 0.5 * (2 / 3) ** 2 > bound > 0.5 * (2 / 3) ** 3


def test_smoothing_sphere_radial_projection():
    """S:417 example: a candidate at distance 2r along +x is projected to anchor + (r, 0, 0); a
    candidate inside the sphere is unchanged."""
    m = oracle.Mesh(points=np.zeros((2, 3), np.float32),
                    anchors=np.array([[0.0, 0.0, 0.0], [2.0, 0.0, 0.0]]),
                    voxel_idx=np.zeros((2, 3), np.int64), quads=np.zeros((0, 4), np.uint32),
                    pairs=np.zeros((0, 2), np.uint32), csr_off=np.array([0, 1, 2], np.uint32),
                    csr_ids=np.array([1, 0], np.uint32), face_mask=np.zeros(2, np.uint8))
    # lambda = 0.5: point 0's candidate is (1, 0, 0) = 2r with d = 0.5 at unit spacing
    out = oracle.smooth(m, (1.0, 1.0, 1.0), 1, 0.5, 0.5, shape=oracle.SPHERE)
    np.testing.assert_array_equal(out[0], [0.5, 0.0, 0.0])
    np.testing.assert_array_equal(out[1], [1.5, 0.0, 0.0])
    out = oracle.smooth(m, (1.0, 1.0, 1.0), 1, 0.5, 10.0, shape=oracle.SPHERE)   # r = 10: inside
    np.testing.assert_array_equal(out[0], [1.0, 0.0, 0.0])


def test_smoothing_sphere_containment_and_large_radius():
    """Containment |p - anchor| <= r on iid data (the sphere binds), and with a radius no point can
    reach the sphere and the box are both inactive: identical trajectories."""
    rng = np.random.default_rng(9)
    a = rng.integers(0, 4, size=(14, 15, 16)).astype(np.uint8)
    sp = (0.8, 1.0, 1.5)
    m = extract(a, spacing=sp)
    d = 0.5
    out = oracle.smooth(m, sp, 10, 0.5, d, shape=oracle.SPHERE)
    dist = np.linalg.norm(out - m.anchors, axis=1)
    r = d * min(sp)
    assert dist.max() <= r * (1 + 1e-12)
    assert np.isclose(dist, r).mean() > 0.01
    big_s = oracle.smooth(m, sp, 10, 0.5, 1e6, shape=oracle.SPHERE)
    big_b = oracle.smooth(m, sp, 10, 0.5, 1e6, shape=oracle.BOX)
    np.testing.assert_array_equal(big_s, big_b)


def test_window_smoothing_matches_full():
    """Windowed oracle (frozen margin layers) reproduces the full oracle on the
    inner layers exactly -- the basis of the full-size sampled parity tests."""
    rng = np.random.default_rng(12)
    n = 14
    a = np.zeros((n, n, n), np.uint16)
    a[1:-1, 1:-1, 1:-1] = rng.integers(0, 3, size=(n - 2, n - 2, n - 2))
    T = 3
    vol = oracle.as_volume(a)
    full = oracle.extract(vol)
    out_full = oracle.smooth(full, (1, 1, 1), T, 0.5, 0.5)
    k0, k1 = 6, 8
    w0, w1 = k0 - T - 1, k1 + T + 1
    P, _, S = oracle.layer_counts(vol)
    base = int(P[:w0].sum())
    win = oracle.extract(oracle.Volume(a[w0 - 1:w1 + 2], vol.dims, w0 - 1), w0, w1, point_base=base)
    lay = win.voxel_idx[:, 2]
    frozen = ((lay == w0) | (lay == w1 - 1)).astype(np.uint8)
    # stencil ids pointing outside the window belong to frozen points only
    out_win = oracle.smooth(win, (1, 1, 1), T, 0.5, 0.5, frozen=frozen)
    sel = (lay >= k0) & (lay < k1)
    gsel = (full.voxel_idx[:, 2] >= k0) & (full.voxel_idx[:, 2] < k1)
    np.testing.assert_array_equal(out_win[sel], out_full[gsel])


# --------------------------------------------------------------------------- triangulation pins
@pytest.mark.parametrize("name", ["triangulate_spec_quad", "triangulate_planar_square"])
def test_triangulation_worked(name):
    case = GOLD[name]
    v = [float(x) for x in case["quad"].split()]
    pts = np.array(v, np.float32).reshape(4, 3)
    tris = oracle.triangulate(np.array([[0, 1, 2, 3]], np.uint32), pts)
    if case["expect_diagonal"] == "02":
        assert tris.tolist() == [[0, 1, 2], [0, 2, 3]]
    else:
        assert tris.tolist() == [[0, 1, 3], [1, 2, 3]]
    assert oracle.triangulate(np.array([[0, 1, 2, 3]], np.uint32), pts, strategy=0).tolist() == [[0, 1, 2], [0, 2, 3]]


def _diag(pts, strategy):
    t = oracle.triangulate(np.array([[0, 1, 2, 3]], np.uint32), np.array(pts, np.float32), strategy=strategy)
    if t.tolist() == [[0, 1, 2], [0, 2, 3]]:
        return "02"
    assert t.tolist() == [[0, 1, 3], [1, 2, 3]]
    return "13"


def test_triangulation_strategies_worked():
    """P:97 names greedy, shortest diagonal, minimum area and most co-planar (reading Q27 for
    the last two).  Expected diagonals by hand arithmetic:
    quad A = (0,0,0),(1,0,0),(1,1,1),(0,1,0): |d02|^2 = 3 > |d13|^2 = 2 -> shortest 13;
      n(a,b,c) = (0,-1,1), n(a,c,d) = (-1,0,1): 2*area 0-2 = 2*sqrt2 = 2.83;
      n(a,b,d) = (0,0,1), n(b,c,d) = (-1,-1,1): 1 + sqrt3 = 2.73 -> min area 13;
      cos 0-2 = 1/2, cos 1-3 = 1/sqrt3 = 0.577 -> most co-planar 13.
    quad B = (2,2,2),(-1,0,0),(2,2,1),(1,2,1): |d02|^2 = 1 < 9 -> shortest 02;
      n(a,b,c) = (2,-3,0), n(a,c,d) = (0,1,0): sqrt13 + 1 = 4.61;
      n(a,b,d) = (2,-1,-2), n(b,c,d) = (0,-1,2): 3 + sqrt5 = 5.24 -> min area 02;
      cos 0-2 = -3/sqrt13 = -0.83, cos 1-3 = -3/(3 sqrt5) = -0.45 -> most co-planar 13.
    Rotating a quad's vertex order by one swaps the roles of the diagonals (same physical
    diagonal chosen); a planar square and a degenerate quad tie -> 0-2 for every strategy."""
    A = [[0, 0, 0], [1, 0, 0], [1, 1, 1], [0, 1, 0]]
    B = [[2, 2, 2], [-1, 0, 0], [2, 2, 1], [1, 2, 1]]
    assert [_diag(A, s) for s in (0, 1, 2, 3)] == ["02", "13", "13", "13"]
    assert [_diag(B, s) for s in (0, 1, 2, 3)] == ["02", "02", "02", "13"]
    flip = {"02": "13", "13": "02"}
    for q in (A, B):
        rot = q[3:] + q[:3]
        for s in (1, 2, 3):
            assert _diag(rot, s) == flip[_diag(q, s)]
    square = [[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]]
    same = [[0.5, 0.5, 0.5]] * 4
    for s in (0, 1, 2, 3):
        assert _diag(square, s) == "02" and _diag(same, s) == "02"


def test_triangulation_count_and_subcycles():
    rng = np.random.default_rng(21)
    a = _random_volume(rng, max_dim=10)
    m = extract(a)
    out = oracle.smooth(m, (1, 1, 1), 5, 0.5, 0.5).astype(np.float32)
    tris = oracle.triangulate(m.quads, out)
    assert len(tris) == 2 * m.n_quads
    for q, (t0, t1) in zip(m.quads.tolist(), tris.reshape(-1, 2, 3).tolist()):
        for t in (t0, t1):
            pos = [q.index(x) for x in t]
            # cyclic subsequence of the quad's cycle (orientation preserved)
            r = pos.index(min(pos))
            rot = pos[r:] + pos[:r]
            assert rot == sorted(rot)
        # the two triangles cover the quad's 4 vertices
        assert set(t0) | set(t1) == set(q)


# --------------------------------------------------------------------------- brute force 3x3x3 (C)
@pytest.mark.slow
def test_bruteforce_all_3x3x3_binary(tmp_path):
    """All 2^27 two-label 3x3x3 volumes against the independent corner/face
    formulation in tests/brute/brute3.c (BASELINE.json north_star)."""
    import os
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    exe = str(tmp_path / "brute3")
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-o", exe,
                           os.path.join(here, "brute", "brute3.c"),
                           os.path.join(os.path.dirname(here), "oracle", "psn_oracle.c"), "-lm"])
    out = subprocess.run([exe, "1"], capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip() == f"ok {1 << 27}"
