"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by
element, on the same seeded inputs.  Extraction outputs must be bit-exact
(points, quads, pairs, CSR offsets/ids, face masks); smoothed coordinates
within 1e-4 x spacing per axis (BASELINE.json north_star); triangles
bit-exact against host triangulation of the GPU's own fp32 points (C-8 i)."""
import numpy as np
import pytest
import torch

import gpu_util as gu
import oracle
import psn_gen

pytestmark = pytest.mark.gpu

TOL = 1e-4   # x spacing, per axis (north_star)


def _corpus(rng, n, max_dim=40):
    out = []
    for t in range(n):
        dims = [int(rng.integers(2, max_dim + 1)) for _ in range(3)]
        if t % 7 == 0:
            dims[0] = int(rng.choice([129, 131, 257, 130]))   # several warps, ragged last chunk
        M, N, O = dims
        dtype = [np.uint8, np.uint16, np.uint32][t % 3]
        kind = t % 4
        if kind == 0:
            a = rng.integers(0, 4, size=(O, N, M))
        elif kind == 1:
            z, y, x = np.meshgrid(np.arange(O), np.arange(N), np.arange(M), indexing="ij")
            c = rng.uniform(0, 1, 3) * np.array([M, N, O])
            r = rng.uniform(1, max(2, min(dims) / 2))
            a = ((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 <= r * r).astype(np.int64) * int(rng.integers(1, 200))
        elif kind == 2:
            a = np.zeros((O, N, M), np.int64)
            a[1:-1, 1:-1, 1:-1] = rng.integers(0, 3, size=(max(O - 2, 0), max(N - 2, 0), max(M - 2, 0)))
        else:
            z, y, x = np.meshgrid(np.arange(O), np.arange(N), np.arange(M), indexing="ij")
            a = (x // int(rng.integers(1, 9)) + 3 * (y // int(rng.integers(1, 9))) + 5 * (z // int(rng.integers(1, 9)))) % 6
        a = a.astype(dtype)
        if dtype == np.uint32 and t % 2:
            a = a * np.uint32(1000003)
        label_set = None
        if t % 5 == 2:
            vals = np.unique(a).tolist()
            label_set = sorted(set(rng.choice(vals, size=max(1, len(vals) // 2)).tolist()) | {0})
        elif t % 5 == 4:
            vals = np.unique(a).tolist()
            label_set = sorted(set(rng.choice(vals, size=max(1, (len(vals) + 1) // 2)).tolist()))
        out.append((a, label_set))
    return out


def _check_volume(a, label_set=None, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0), T=5):
    p, vol, mesh, dev = gu.gpu_extract(a, spacing, origin, label_set)
    om = oracle.extract(oracle.as_volume(a, spacing, origin, label_set))
    g = gu.mesh_np(mesh)
    assert (mesh.n_points, mesh.n_quads, mesh.n_stencil) == (om.n_points, om.n_quads, om.n_stencil)
    gu.assert_mesh_equal(g, om)
    counts, trims = p.rows(vol, mesh.ws)
    gu.check_rows(counts.cpu().numpy().view(np.uint32), trims.cpu().numpy(), om,
                  oracle.as_volume(a, spacing, origin, label_set))
    if om.n_points:
        pts = p.smooth(vol, mesh, T, 0.5, 0.5)
        ref = oracle.smooth(om, spacing, T, 0.5, 0.5)
        # 1e-4 x spacing, plus the fp32 output's single rounding (half an ulp, which alone exceeds
        # 1e-4 once |coordinate| > 2048 x spacing -- the wide-row cases; every BASELINE config is below)
        gp64 = pts[:om.n_points].cpu().numpy().astype(np.float64)
        half_ulp = 0.5 * np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
        err = (np.abs(gp64 - ref) - half_ulp) / np.array(spacing)
        assert err.max() <= TOL, err.max()
        # containment: |p - anchor| <= d*s + ulp32 of the fp32 output (its one rounding)
        gp = pts[:om.n_points].cpu().numpy()
        dev_ = np.abs(gp.astype(np.float64) - om.anchors)
        ulp = np.spacing(np.maximum(np.abs(om.points), np.abs(gp)).astype(np.float32)).astype(np.float64)
        assert np.all(dev_ <= 0.5 * np.array(spacing) + ulp)
        if om.n_quads:
            tris = p.triangulate(mesh, pts)
            host = oracle.triangulate(om.quads, pts[:om.n_points].cpu().numpy())
            np.testing.assert_array_equal(gu.u32(tris, 2 * om.n_quads), host)
    return mesh


@pytest.mark.parametrize("counting,emission", [(0, 0), (1, 0), (0, 2), (1, 2)])
def test_random_corpus_bit_exact(counting, emission):
    """Every counting kernel (0 = warp-per-row k_count3, 1 = x-tiled k_count) and emission kernel
    (0 = band-staged, 2 = general scan-based) reproduces the oracle bit for bit."""
    p = gu.psn()
    rng = np.random.default_rng(20240126)
    try:
        p.set_counting(counting)
        p.set_emission(emission)
        for a, ls in _corpus(rng, 120):
            _check_volume(a, ls, spacing=(0.8, 1.0, 1.5), origin=(-3.0, 2.0, 10.0))
    finally:
        p.set_counting(0)
        p.set_emission(0)


@pytest.mark.parametrize("dense", ["-1", "0", "1"])
def test_emission_density_variants_bit_exact(monkeypatch, dense):
    """k_emit_band's two density variants (STG: dense rounds staged through shared memory, or not)
    and the dual launch (both variants, the scan totals pick one on the device) reproduce the
    oracle bit for bit on sparse and dense (i.i.d., > 4.7 stencil entries per point) meshes,
    whichever the host selects -- including the wrong one for the mesh's density."""
    monkeypatch.setenv("PSN_EMIT_DENSE", dense)
    rng = np.random.default_rng(5150)
    for a, ls in _corpus(rng, 24):
        _check_volume(a, ls, spacing=(0.8, 1.0, 1.5), origin=(-3.0, 2.0, 10.0), T=2)
    iid = rng.integers(0, 4, size=(20, 37, 131)).astype(np.uint8)
    mesh = _check_volume(iid, T=2)
    assert mesh.n_stencil * 32 >= 150 * mesh.n_points   # dense: the staging variant's case


def test_two_by_two_by_two_exhaustive():
    """All 2^8 binary and 3^8 ternary 2x2x2 volumes in one batch each (as slabs of one volume
    would mix them; here each is its own call through the ABI)."""
    p = gu.psn()
    for nval in (2, 3):
        import itertools
        for vals in itertools.product(range(nval), repeat=8):
            a = np.array(vals, np.uint8).reshape(2, 2, 2)
            _, vol, mesh, _ = gu.gpu_extract(a)
            om = oracle.extract(oracle.as_volume(a))
            assert (mesh.n_points, mesh.n_quads, mesh.n_stencil) == (om.n_points, om.n_quads, om.n_stencil)
            if om.n_points:
                gu.assert_mesh_equal(gu.mesh_np(mesh), om)
    del p


def test_iid_contains_every_2x2x2_pattern():
    """Large iid volumes contain every 2x2x2 pattern thousands of times."""
    rng = np.random.default_rng(5)
    for dtype, M in ((np.uint8, 96), (np.uint16, 100), (np.uint32, 64)):
        a = rng.integers(0, 3, size=(40, 37, M)).astype(dtype)
        _check_volume(a, T=10)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_config_full(name):
    spec = psn_gen.config(name)
    dev = psn_gen.generate_device(spec)
    host = psn_gen.generate_host(spec)
    np.testing.assert_array_equal(dev.cpu().numpy(), host)
    T, lam, d = psn_gen.SMOOTHING[name]
    sp = tuple(spec.spacing)
    p = gu.psn()
    vol = p.volume(dev, spacing=sp)
    mesh = p.extract(vol)
    om = oracle.extract(oracle.as_volume(host, sp))
    gu.assert_mesh_equal(gu.mesh_np(mesh), om)
    counts, trims = p.rows(vol, mesh.ws)
    gu.check_rows(counts.cpu().numpy().view(np.uint32), trims.cpu().numpy(), om, oracle.as_volume(host, sp))
    pts = p.smooth(vol, mesh, T, lam, d)
    ref = oracle.smooth(om, sp, T, lam, d)
    gp = pts[:om.n_points].cpu().numpy()
    err = np.abs(gp.astype(np.float64) - ref) / np.array(sp)
    assert err.max() <= TOL, err.max()
    tris = p.triangulate(mesh, pts)
    np.testing.assert_array_equal(gu.u32(tris, 2 * om.n_quads), oracle.triangulate(om.quads, gp))
    # C-8 (ii): against the fp64 oracle, differences only on near-ties
    tref = oracle.triangulate(om.quads, ref.astype(np.float32))
    diff = np.nonzero((gu.u32(tris, 2 * om.n_quads) != tref).any(1))[0] // 2
    tau = TOL * max(sp)
    for q in np.unique(diff):
        v = om.quads[q]
        d02 = np.linalg.norm(ref[v[2]] - ref[v[0]]); d13 = np.linalg.norm(ref[v[3]] - ref[v[1]])
        assert abs(d02 ** 2 - d13 ** 2) <= 4 * np.sqrt(3) * tau * (d02 + d13) + 24 * tau ** 2


def test_fused_count_emit_matches_two_phase():
    spec = psn_gen.config("c2")
    dev = psn_gen.generate_device(spec)
    p = gu.psn()
    vol = p.volume(dev)
    ref = p.extract(vol)
    g0 = gu.mesh_np(ref)
    mesh = p.alloc_mesh(ref.n_window, ref.n_points, ref.n_quads, ref.n_stencil)
    ws = p.workspace(vol)
    lab = p.labels(None)
    for _ in range(2):
        p.extract_into(vol, lab, ws, mesh)
        p.totals(vol, ws, mesh)
        g = gu.mesh_np(mesh)
        for k in g0:
            np.testing.assert_array_equal(g[k], g0[k])
    # too small capacity: the fused path skips emission and reports it
    small = p.alloc_mesh(ref.n_window - 1, ref.n_points, ref.n_quads, ref.n_stencil)
    p.extract_into(vol, lab, ws, small)
    from paper_2401_14906_b200.psn import PSNError, PSN_ERR_CAPACITY
    with pytest.raises(PSNError) as e:
        p.totals(vol, ws, small)
    assert e.value.status == PSN_ERR_CAPACITY


def test_deterministic_repeats():
    rng = np.random.default_rng(9)
    a = rng.integers(0, 4, size=(30, 33, 70)).astype(np.uint16)
    outs = [gu.mesh_np(gu.gpu_extract(a)[2]) for _ in range(3)]
    for o in outs[1:]:
        for k in o:
            np.testing.assert_array_equal(o[k], outs[0][k])


def test_degenerate_and_errors():
    from paper_2401_14906_b200.psn import PSNError, PSN_ERR_ARG, PSN_ERR_LABELS
    p = gu.psn()
    for a in (np.zeros((8, 8, 8), np.uint8), np.full((8, 8, 8), 7, np.uint16), np.zeros((2, 2, 2), np.uint8)):
        _, _, mesh, _ = gu.gpu_extract(a)
        assert (mesh.n_points, mesh.n_quads, mesh.n_stencil) == (0, 0, 0)
        assert int(mesh.stencil_offsets[0]) == 0
    dev = torch.zeros((1, 4, 4), dtype=torch.uint8, device="cuda")
    with pytest.raises(PSNError) as e:
        p.extract(p.volume(dev))          # O = 1 < 2
    assert e.value.status == PSN_ERR_ARG
    dev = torch.zeros((4, 4, 4), dtype=torch.uint8, device="cuda")
    with pytest.raises(PSNError) as e:
        p.extract(p.volume(dev), label_set=[])
    assert e.value.status == PSN_ERR_LABELS
    with pytest.raises(PSNError) as e:
        p.extract(p.volume(dev), label_set=[0xFFFFFFFF])
    assert e.value.status == PSN_ERR_LABELS
    with pytest.raises(PSNError) as e:
        p.extract(p.volume(dev, spacing=(1.0, 0.0, 1.0)))
    assert e.value.status == PSN_ERR_ARG
    _, vol, mesh, _ = gu.gpu_extract(np.pad(np.ones((2, 2, 2), np.uint8), 2))
    with pytest.raises(PSNError) as e:
        p.smooth(vol, mesh, 3, 1.5, 0.5)
    assert e.value.status == PSN_ERR_ARG
    for fn, bad in ((p.set_counting, 2), (p.set_emission, 1), (p.set_constraint, 2), (p.set_smoothing, 5)):
        with pytest.raises(PSNError) as e:
            fn(bad)
        assert e.value.status == PSN_ERR_ARG
    with pytest.raises(PSNError) as e:
        p.triangulate(mesh, mesh.points, strategy=4)
    assert e.value.status == PSN_ERR_ARG
    # float4 offset buffers must be 16-byte aligned
    ws = p.smooth_workspace(mesh)
    p.smooth_prepare(vol, mesh, ws)
    flat = torch.zeros(4 * mesh.n_window + 1, dtype=torch.float32, device="cuda")
    with pytest.raises(PSNError) as e:
        p.smooth_step(vol, mesh, ws, None, flat[1:].view(-1, 4), 0.5, 0.5)
    assert e.value.status == PSN_ERR_ARG


def test_smoothing_zero_iterations_is_anchors():
    rng = np.random.default_rng(2)
    a = rng.integers(0, 3, size=(12, 13, 17)).astype(np.uint8)
    p, vol, mesh, _ = gu.gpu_extract(a, spacing=(0.8, 0.8, 1.5), origin=(5.0, -1.0, 0.25))
    pts = p.smooth(vol, mesh, 0, 0.5, 0.5)
    np.testing.assert_array_equal(pts[:mesh.n_points].cpu().numpy(), mesh.points[:mesh.n_points].cpu().numpy())
    pts = p.smooth(vol, mesh, 4, 0.0, 0.5)
    np.testing.assert_array_equal(pts[:mesh.n_points].cpu().numpy(), mesh.points[:mesh.n_points].cpu().numpy())


def test_wide_rows_multi_xtile():
    """M > 1024 splits rows over several CTAs (global-atomic row counters)."""
    rng = np.random.default_rng(77)
    a = rng.integers(0, 3, size=(4, 5, 1500)).astype(np.uint16)
    _check_volume(a, T=3)
    a = np.zeros((5, 6, 2100), np.uint8)
    a[2, 2:4, 1000:1100] = 3
    _check_volume(a, T=3)
    # u32 rows wider than one k_count x-tile (1024): general (scan-based) k_emit path
    a = rng.integers(0, 3, size=(4, 5, 1500)).astype(np.uint32)
    _check_volume(a, T=3)
    a = rng.integers(0, 3, size=(3, 4, 4500)).astype(np.uint8)
    _check_volume(a, T=2)


@pytest.mark.parametrize("G,tile", [(0, 0), (1, 256), (3, 512), (7, 2048)])
def test_wavefront_smoothing_bit_identical(G, tile):
    """psn_smooth's wavefront (temporally blocked) schedule == one launch per iteration, bit for bit,
    and within 1e-4 x spacing of the fp64 oracle."""
    p = gu.psn()
    rng = np.random.default_rng(31 + G)
    vols = [rng.integers(0, 4, size=(30, 40, 50)).astype(np.uint8),
            psn_gen.generate_host(psn_gen.config("c2"))[:80]]
    try:
        for a in vols:
            _, vol, mesh, _ = gu.gpu_extract(a, spacing=(0.8, 1.0, 1.5))
            T = 11
            ws = p.smooth_workspace(mesh)
            p.set_smoothing(1, 0)
            ref = p.smooth(vol, mesh, T, 0.5, 0.5, ws=ws).clone()
            p.set_smoothing(0, G, tile)
            out = p.smooth(vol, mesh, T, 0.5, 0.5, ws=ws)
            p.smooth_status(mesh, ws)
            np.testing.assert_array_equal(out[:mesh.n_points].cpu().numpy(), ref[:mesh.n_points].cpu().numpy())
            om = oracle.extract(oracle.as_volume(a, (0.8, 1.0, 1.5)))
            o64 = oracle.smooth(om, (0.8, 1.0, 1.5), T, 0.5, 0.5)
            err = np.abs(out[:mesh.n_points].cpu().numpy().astype(np.float64) - o64) / np.array((0.8, 1.0, 1.5))
            assert err.max() <= TOL
    finally:
        p.set_smoothing(1, 0, 0)


@pytest.mark.parametrize("shape", [0, 1])
def test_step_loop_matches_psn_smooth(shape):
    """psn_smooth_prepare + T x psn_smooth_step (+ finalize), the slab path on a whole
    volume, gives psn_smooth's bits for the box and the sphere constraint."""
    p = gu.psn()
    rng = np.random.default_rng(55)
    a = rng.integers(0, 3, size=(14, 17, 23)).astype(np.uint8)
    _, vol, mesh, _ = gu.gpu_extract(a, spacing=(0.8, 1.0, 1.5))
    try:
        p.set_constraint(shape)
        T = 8
        ws = p.smooth_workspace(mesh)
        ref = p.smooth(vol, mesh, T, 0.5, 0.5, ws=ws).clone()
        p.smooth_prepare(vol, mesh, ws)
        bufs = [p.offsets_buffer(mesh.n_window, "cuda") for _ in range(2)]
        src = None
        for t in range(T):
            p.smooth_step(vol, mesh, ws, src, bufs[t & 1], 0.5, 0.5)
            src = bufs[t & 1]
        out = torch.empty_like(ref)
        p.smooth_finalize(vol, mesh, src, out)
        n = mesh.n_points
        assert torch.equal(out[:n], ref[:n])
    finally:
        p.set_constraint(0)


def test_packed_smoothing_cache_bit_identical(monkeypatch):
    """The packed 8-byte smoothing cache (id distances, chosen when M-1 < 2^10 and
    (M-1)(N-1) < 2^21) gives the same bits as the 16-byte one, including a volume at
    the packing limits (rows of 1023 cells: y distances up to 1022; dense layers)."""
    p = gu.psn()
    rng = np.random.default_rng(77)
    vols = [rng.integers(0, 4, size=(12, 40, 60)).astype(np.uint8),
            rng.integers(0, 3, size=(4, 9, 1024)).astype(np.uint16),
            psn_gen.generate_host(psn_gen.config("c2"))[100:140]]
    for a in vols:
        dev = torch.from_numpy(np.ascontiguousarray(a)).cuda()
        vol = p.volume(dev, spacing=(0.8, 1.0, 1.5))
        labels, ws_e = p.labels(None), p.workspace(vol)
        counted = p.count(vol, labels, ws_e)
        mesh = p.alloc_mesh(counted.n_points, counted.n_points, counted.n_quads, counted.n_stencil, smooth_cache=True)
        mesh = p.emit(vol, labels, ws_e, counted, mesh=mesh)
        assert mesh.c.smooth_cache_valid == 1          # written by the emission (band kernel, packable dims)
        ws = p.smooth_workspace(mesh)
        packed = p.smooth(vol, mesh, 9, 0.5, 0.5, ws=ws).clone()   # uses the emission's cache
        mesh.c.smooth_cache_valid = 0
        prep = p.smooth(vol, mesh, 9, 0.5, 0.5, ws=ws).clone()     # k_smooth_prep8 builds it from the CSR
        mesh.c.smooth_cache_valid = 1
        monkeypatch.setenv("PSN_SMOOTH_NBR16", "1")
        wide = p.smooth(vol, mesh, 9, 0.5, 0.5, ws=ws)
        monkeypatch.delenv("PSN_SMOOTH_NBR16")
        n = mesh.n_points
        assert torch.equal(packed[:n], prep[:n])
        assert torch.equal(packed[:n], wide[:n])
        # the emitted cache equals the one the prep kernel builds (same bits)
        ws2 = p.smooth_workspace(mesh)
        p.smooth_prepare(vol, mesh, ws2)
        built = ws2[:8 * n].view(torch.int32).view(n, 2)
        assert torch.equal(built, mesh.smooth_cache[:n])


@pytest.mark.parametrize("sphere", [0, 1])
def test_split_smoothing_cache_bit_identical(monkeypatch, sphere):
    """Iterations 2..T with the split cache (k_smooth_split: the packed entry's lo word in the
    offsets' w slot, the hi word in a 4-byte array) give the same bits as k_smooth_v4 reading
    the 8-byte entries every iteration -- emitted cache, prep-built cache, and the cache built
    by the first iteration itself (k_smooth_first), and iterations 1 + 2 in one pass from the face
    masks (k_smooth_first2); T = 1, 2, 3, 9, box and sphere constraints,
    and a mesh too small for the split (it falls back)."""
    p = gu.psn()
    rng = np.random.default_rng(91)
    vols = [rng.integers(0, 4, size=(12, 40, 60)).astype(np.uint8),
            psn_gen.generate_host(psn_gen.config("c2"))[96:150],
            np.pad(np.ones((1, 1, 1), np.uint16), 1)]
    p.set_constraint(sphere)
    try:
        for a in vols:
            dev = torch.from_numpy(np.ascontiguousarray(a)).cuda()
            vol = p.volume(dev, spacing=(0.8, 1.0, 1.5))
            labels, ws_e = p.labels(None), p.workspace(vol)
            counted = p.count(vol, labels, ws_e)
            mesh = p.alloc_mesh(counted.n_points, counted.n_points, counted.n_quads, counted.n_stencil,
                                smooth_cache=True)
            mesh = p.emit(vol, labels, ws_e, counted, mesh=mesh)
            ws = p.smooth_workspace(mesh)
            n = mesh.n_points
            for T in (1, 2, 3, 9):
                for cached in (1, 0):
                    mesh.c.smooth_cache_valid = cached
                    split = p.smooth(vol, mesh, T, 0.5, 0.5, ws=ws).clone()   # cached=0: k_smooth_first2
                    monkeypatch.setenv("PSN_SMOOTH_NOFIRST2", "1")
                    split1 = p.smooth(vol, mesh, T, 0.5, 0.5, ws=ws).clone()  # k_smooth_first + split
                    monkeypatch.delenv("PSN_SMOOTH_NOFIRST2")
                    monkeypatch.setenv("PSN_SMOOTH_NOFIRST", "1")
                    split_prep = p.smooth(vol, mesh, T, 0.5, 0.5, ws=ws).clone()   # k_smooth_prep8 + split
                    monkeypatch.delenv("PSN_SMOOTH_NOFIRST")
                    monkeypatch.setenv("PSN_SMOOTH_NOSPLIT", "1")
                    plain = p.smooth(vol, mesh, T, 0.5, 0.5, ws=ws)
                    monkeypatch.delenv("PSN_SMOOTH_NOSPLIT")
                    assert torch.equal(split[:n], plain[:n]), (a.shape, T, cached)
                    assert torch.equal(split_prep[:n], plain[:n]), (a.shape, T, cached)
                    assert torch.equal(split1[:n], plain[:n]), (a.shape, T, cached)
                mesh.c.smooth_cache_valid = 1
    finally:
        p.set_constraint(0)


def test_dense_wide_rows_and_layers_smoothing():
    """Dense iid volumes whose rows hold ~1400 points and whose layers hold ~600K points, so
    stencil neighbours are far apart in id space: extraction and smoothing still match the oracle."""
    rng = np.random.default_rng(123)
    a = rng.integers(0, 4, size=(4, 6, 1500)).astype(np.uint16)
    _check_volume(a, T=3)
    a = rng.integers(0, 4, size=(3, 820, 820)).astype(np.uint8)
    _check_volume(a, T=2)


@pytest.mark.parametrize("spacing", [(1.0, 1.0, 1.0), (0.8, 0.8, 1.5)])
def test_sphere_constraint_smoothing(spacing):
    """psn_smooth with the sphere constraint (reading Q26) against the fp64 oracle: within
    1e-4 x spacing, and every point within d*min(s) of its voxel centre (+ fp32 rounding); the
    per-iteration and wavefront schedules stay bit-identical."""
    p = gu.psn()
    rng = np.random.default_rng(61)
    vols = [rng.integers(0, 4, size=(17, 19, 23)).astype(np.uint8),
            psn_gen.generate_host(psn_gen.config("c1")),
            np.pad(np.ones((5, 5, 5), np.uint16), 2)]
    try:
        p.set_constraint(1)
        for a in vols:
            _, vol, mesh, _ = gu.gpu_extract(a, spacing=spacing, origin=(3.0, -1.0, 0.5))
            om = oracle.extract(oracle.as_volume(a, spacing, (3.0, -1.0, 0.5)))
            for T in (1, 4, 12):
                out = p.smooth(vol, mesh, T, 0.5, 0.5)
                ref = oracle.smooth(om, spacing, T, 0.5, 0.5, shape=oracle.SPHERE)
                g = out[:om.n_points].cpu().numpy().astype(np.float64)
                err = np.abs(g - ref) / np.array(spacing)
                assert err.max() <= TOL, (T, err.max())
                r = 0.5 * min(spacing)
                dist = np.linalg.norm(g - om.anchors, axis=1)
                assert dist.max() <= r + 4 * np.spacing(np.float32(np.abs(g).max())), dist.max() - r
            ws = p.smooth_workspace(mesh)
            ref = p.smooth(vol, mesh, 9, 0.5, 0.5, ws=ws).clone()
            p.set_smoothing(0, 3, 256)
            out = p.smooth(vol, mesh, 9, 0.5, 0.5, ws=ws)
            p.smooth_status(mesh, ws)
            p.set_smoothing(1, 0, 0)
            np.testing.assert_array_equal(out[:mesh.n_points].cpu().numpy(), ref[:mesh.n_points].cpu().numpy())
    finally:
        p.set_constraint(0)
        p.set_smoothing(1, 0, 0)


@pytest.mark.parametrize("strategy", [0, 1, 2, 3])
def test_triangulation_strategies(strategy):
    """k_triangulate for fixed / shortest / minimum-area / most-co-planar (reading Q27):
    bit-exact against the host triangulation of the same fp32 points (C-8 i), on smoothed
    meshes (non-planar quads) and on the unsmoothed voxel-centre mesh (planar quads: ties)."""
    rng = np.random.default_rng(71)
    for a in (rng.integers(0, 3, size=(15, 16, 17)).astype(np.uint16), psn_gen.generate_host(psn_gen.config("c1"))):
        p, vol, mesh, _ = gu.gpu_extract(a, spacing=(0.8, 1.0, 1.5))
        om = oracle.extract(oracle.as_volume(a, (0.8, 1.0, 1.5)))
        for pts in (p.smooth(vol, mesh, 6, 0.5, 0.5), mesh.points):
            tris = p.triangulate(mesh, pts, strategy=strategy)
            host = oracle.triangulate(om.quads, pts[:om.n_points].cpu().numpy(), strategy=strategy)
            np.testing.assert_array_equal(gu.u32(tris, 2 * om.n_quads), host)


def test_surface_nets_stream_matches_single_calls():
    """SurfaceNetsStream (pipelined host-buffer API: copy / compute / readback streams, rotating
    slots) returns, for every submitted volume, exactly the outputs of a plain extraction +
    smoothing of that volume, also when consecutive volumes differ."""
    from paper_2401_14906_b200.psn import SurfaceNetsStream
    p = gu.psn()
    rng = np.random.default_rng(99)
    base = psn_gen.generate_host(psn_gen.config("c1"))
    big = np.zeros_like(base)
    big[2:-2, 2:-2, 2:-2] = rng.integers(0, 3, size=(28, 28, 28))   # larger totals: slot buffers grow
    vols = [base, np.roll(base, 3, axis=2), big, np.flip(base, 1).copy(), base, big]
    sp = (0.8, 1.0, 1.5)
    T, lam, d = 7, 0.5, 0.5
    sns = SurfaceNetsStream(p, base.shape, torch.uint16, sp, T, lam, d, depth=2)
    tickets, expected = [], []
    for a in vols:
        h = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        tickets.append(sns.submit(h))
        _, vol, mesh, _ = gu.gpu_extract(a, spacing=sp)
        pts = p.smooth(vol, mesh, T, lam, d)
        expected.append((pts[:mesh.n_points].cpu().numpy(), gu.u32(mesh.quads, mesh.n_quads), gu.u32(mesh.pairs, mesh.n_quads)))
        if len(tickets) >= 2:
            t = tickets[-2]
            pts_h, q_h, pr_h = sns.result(t)
            e = expected[-2]
            np.testing.assert_array_equal(pts_h.numpy(), e[0])
            np.testing.assert_array_equal(q_h.numpy().view(np.uint32), e[1])
            np.testing.assert_array_equal(pr_h.numpy().view(np.uint32), e[2])
    pts_h, q_h, pr_h = sns.result(tickets[-1])
    np.testing.assert_array_equal(pts_h.numpy(), expected[-1][0])
    np.testing.assert_array_equal(q_h.numpy().view(np.uint32), expected[-1][1])


@pytest.mark.parametrize("name", ["c1", "c5b"])
def test_pipeline_graph_replay_identical(name):
    """bench.py replays the steady-state step as two CUDA graphs (Pipeline.capture): the replayed
    extraction + smoothing (+ triangulation) write exactly what the direct library calls write."""
    from paper_2401_14906_b200.psn import Pipeline
    spec = psn_gen.config(name)
    T, lam, d = psn_gen.SMOOTHING[name]
    p = gu.psn()
    labels = psn_gen.generate_device(spec)
    vol = p.volume(labels, spacing=tuple(spec.spacing))
    pipe = Pipeline(p, vol, T, lam, d, triangulate=True)
    pipe.run()
    torch.cuda.synchronize()
    m = pipe.mesh
    P, Q, S = pipe.counts
    ref = [t.clone() for t in (m.points[:P], m.quads[:Q], m.pairs[:Q], m.stencil_offsets[:P + 1],
                               m.stencil_ids[:S], m.face_masks[:P], pipe.out[:P], pipe.tris[:2 * Q])]
    for t in (m.points, m.quads, m.stencil_ids, pipe.out, pipe.tris):
        t.zero_()
    pipe.capture()
    for t in (m.points, m.quads, m.stencil_ids, pipe.out, pipe.tris):
        t.zero_()
    pipe.replay_extract()
    pipe.replay_smooth()
    torch.cuda.synchronize()
    assert pipe.check()
    got = (m.points[:P], m.quads[:Q], m.pairs[:Q], m.stencil_offsets[:P + 1], m.stencil_ids[:S], m.face_masks[:P],
           pipe.out[:P], pipe.tris[:2 * Q])
    for a_, b_ in zip(ref, got):
        assert torch.equal(a_, b_)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.uint32])
def test_row_width_class_boundaries(dtype):
    """Row widths at the edges of the compile-time classes: k_count3's FULL rows (exactly 32*CPL
    16-byte chunks, CPL = 1, 2, 4) and k_emit_band's 16 / 32 plane words, one element either side,
    plus one-voxel rows (M = 2) and two-row / two-layer volumes -- bit-exact vs the oracle."""
    rng = np.random.default_rng(int(np.dtype(dtype).itemsize) * 101)
    E = 16 // np.dtype(dtype).itemsize
    widths = {2, 3, 33, 34, 512, 513, 514, 1024, 1025, 1026}
    for cpl in (1, 2, 4):
        full = 32 * cpl * E
        widths |= {full - E + 2, full + 1, full + 2}        # M - 1 = smallest / largest FULL, and one past
    for M in sorted(w for w in widths if w * np.dtype(dtype).itemsize <= 8192 and w >= 2):
        for (N, O) in ((5, 4), (2, 3), (3, 2)):
            a = rng.integers(0, 3, size=(O, N, M)).astype(dtype)
            if dtype == np.uint32:
                a = a * np.uint32(0x10001)
            _check_volume(a, T=2)


@pytest.mark.parametrize("dtype,M", [(np.uint16, 257), (np.uint8, 131), (np.uint8, 262), (np.uint16, 130),
                                     (np.uint32, 129)])
def test_unaligned_rows_staging(dtype, M):
    """Rows whose byte length is not a multiple of 16 (k_count3 cannot TMA them as they are): odd
    1- / 2-byte lengths go through the aligned-superset staging + shared-memory shift, 4- / 8-byte
    multiples through cp.async words -- several j-blocks and ring wrap-arounds, bit-exact vs the oracle."""
    rng = np.random.default_rng(M)
    O, N = 30, 41
    z, y, x = np.meshgrid(np.arange(O), np.arange(N), np.arange(M), indexing="ij")
    a = np.zeros((O, N, M), np.int64)
    for lab in range(1, 6):
        c = rng.uniform(0, 1, 3) * np.array([M, N, O])
        r = rng.uniform(6, 18)
        a[(x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 <= r * r] = lab
    m = rng.random(a.shape) < 0.01
    a[m] = rng.integers(0, 6, int(m.sum()))
    _check_volume(a.astype(dtype), T=3)


def test_volume_keeps_its_labels_alive():
    """PSN.volume holds the label tensor: a volume built from a temporary stays valid after the
    temporary's last Python reference is dropped and its memory would otherwise be reused."""
    import gc
    rng = np.random.default_rng(11)
    a = rng.integers(0, 3, size=(20, 24, 28)).astype(np.uint16)
    p = gu.psn()
    vol = p.volume(torch.from_numpy(a).cuda())   # no other reference to the device tensor
    gc.collect()
    junk = torch.full((4 << 20,), 0x5A5A, dtype=torch.int32, device="cuda")   # would overwrite freed memory
    mesh = p.extract(vol)
    torch.cuda.synchronize()
    om = oracle.extract(oracle.as_volume(a))
    assert (mesh.n_points, mesh.n_quads, mesh.n_stencil) == (om.n_points, om.n_quads, om.n_stencil)
    assert np.array_equal(gu.u32(mesh.quads, mesh.n_quads), om.quads)
    del junk
