"""Full-size parity at BASELINE.json's configs (c3, c4, c5a, c5b) and the NEXT-1 config c6, in the launch
configuration bench.py times (psn.Pipeline: PSN_COUNT|PSN_EMIT with preallocated capacities, then
psn_smooth).  EVERY layer is compared:

  * per-layer and per-row plan: the GPU's per-voxel-row P/Q/S counts (psn_extract_rows) summed per
    layer equal the oracle's per-layer counts over the whole volume; per row they equal the counts of
    the oracle's emitted mesh, and the GPU's row trims are the tight point ranges, inside the
    paper's trim-derived voxel-row range;
  * every array, bit for bit: the oracle extracts contiguous layer blocks [k0, k1) with global ids
    (point_base / stencil_base from its own per-layer counts) in a thread pool, and each block is
    compared with the matching slices of the GPU arrays -- the blocks tile all layers;
  * smoothing: >= 8 two-layer windows spread over z, both ends included; the oracle smooths each window
    extended by T+1 frozen layers per side (errors from a frozen layer travel one stencil hop per
    iteration, so the inner layers are exact -- pinned on CPU by test_window_smoothing_matches_full);
    GPU within 1e-4 x spacing (every coordinate of these configs is < 2048 x spacing, so no
    half-ulp allowance is needed, reading Q28).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import gpu_util as gu
import oracle
import psn_gen
from paper_2401_14906_b200.psn import Pipeline

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL = 1e-4
NT = max(2, min(os.cpu_count() or 8, 48))


def pmap(fn, items):
    with ThreadPoolExecutor(NT) as ex:
        return list(ex.map(fn, items))


def layer_counts_parallel(vol, nthreads=NT):
    O = vol.dims[2]
    nl = O - 1
    bounds = [(i * nl // nthreads, (i + 1) * nl // nthreads) for i in range(nthreads)]
    parts = pmap(lambda b: oracle.layer_counts(vol, b[0], b[1]), bounds)
    return tuple(np.concatenate([p[i] for p in parts]) for i in range(3))


@pytest.fixture(scope="module", params=["c3", "c5b", "c5a", "c4", "c6"])
def run(request):
    name = request.param
    spec = psn_gen.config(name)
    T, lam, d = psn_gen.SMOOTHING[name]
    sp = tuple(spec.spacing)
    p = gu.psn()
    labels = psn_gen.generate_device(spec)
    vol = p.volume(labels, spacing=sp)
    pipe = Pipeline(p, vol, T, lam, d)
    pipe.run()             # bench's steady-state step
    torch.cuda.synchronize()
    assert pipe.check()
    counts, trims = p.rows(vol, pipe.ws)
    counts = counts.cpu().numpy().view(np.uint32)
    trims = trims.cpu().numpy()
    host = labels.cpu().numpy()
    ovol = oracle.Volume(host, (spec.M, spec.N, spec.O), 0, sp)
    Pl, Ql, Sl = layer_counts_parallel(ovol)
    yield dict(name=name, spec=spec, pipe=pipe, host=host, ovol=ovol, Pl=Pl, Ql=Ql, Sl=Sl, T=T, lam=lam, d=d, sp=sp,
               counts=counts, trims=trims)
    del pipe, labels
    torch.cuda.empty_cache()


def test_totals_and_layer_counts(run):
    pipe, spec = run["pipe"], run["spec"]
    assert pipe.counts == (int(run["Pl"].sum()), int(run["Ql"].sum()), int(run["Sl"].sum()))
    per_layer = run["counts"].astype(np.int64).reshape(3, spec.O - 1, spec.N - 1).sum(-1)
    np.testing.assert_array_equal(per_layer[0], run["Pl"])
    np.testing.assert_array_equal(per_layer[1], run["Ql"])
    np.testing.assert_array_equal(per_layer[2], run["Sl"])


def _blocks(nl, n):
    n = max(1, min(n, nl))
    return [(i * nl // n, (i + 1) * nl // n) for i in range(n) if (i + 1) * nl // n > i * nl // n]


def test_all_layers_bit_exact(run):
    """Every array of every layer, bit for bit, plus the per-row plan and trims."""
    pipe, spec = run["pipe"], run["spec"]
    m = pipe.mesh
    nl, NV = spec.O - 1, spec.N - 1
    Pc = np.r_[0, np.cumsum(run["Pl"])]
    Qc = np.r_[0, np.cumsum(run["Ql"])]
    Sc = np.r_[0, np.cumsum(run["Sl"])]
    blocks = _blocks(nl, max(4 * NT, nl // 16))

    def work(b):
        k0, k1 = b
        pb, qb, sb = int(Pc[k0]), int(Qc[k0]), int(Sc[k0])
        om = oracle.extract(run["ovol"], k0, k1, point_base=pb, stencil_base=sb)
        P, Q, S = om.n_points, om.n_quads, om.n_stencil
        assert (P, Q, S) == (int(Pc[k1]) - pb, int(Qc[k1]) - qb, int(Sc[k1]) - sb)
        np.testing.assert_array_equal(m.points[pb:pb + P].cpu().numpy(), om.points)
        np.testing.assert_array_equal(m.quads[qb:qb + Q].cpu().numpy().view(np.uint32), om.quads)
        np.testing.assert_array_equal(m.pairs[qb:qb + Q].cpu().numpy().view(np.uint32), om.pairs)
        np.testing.assert_array_equal(m.stencil_offsets[pb:pb + P + 1].cpu().numpy().view(np.uint32), om.csr_off)
        np.testing.assert_array_equal(m.stencil_ids[sb:sb + S].cpu().numpy().view(np.uint32), om.csr_ids)
        np.testing.assert_array_equal(m.face_masks[pb:pb + P].cpu().numpy(), om.face_mask)
        r0, r1 = NV * k0, NV * k1
        gu.check_rows(run["counts"][:, r0:r1], run["trims"][r0:r1], om, run["ovol"], k0, k1)
        return k1 - k0

    covered = sum(pmap(work, blocks))
    assert covered == nl                      # the blocks tile every voxel layer


def test_smoothing_windows(run):
    """>= 8 two-layer windows, evenly spread over z and including both ends, plus three at point quantiles."""
    pipe, spec, T = run["pipe"], run["spec"], run["T"]
    nl = spec.O - 1
    Pl = run["Pl"]
    even = sorted(set(np.linspace(0, nl - 2, 8).round().astype(int).tolist()))
    assert len(even) == 8 and even[0] == 0 and even[-1] == nl - 2
    # plus windows at the 10/50/90 % quantiles of the points (c5b's one small sphere misses every even window)
    cum = np.cumsum(Pl)
    quant = [min(int(np.searchsorted(cum, q * cum[-1])), nl - 2) for q in (0.1, 0.5, 0.9)]
    starts = sorted(set(even + quant))

    def work(k0):
        k1 = k0 + 2
        wa, wb = max(0, k0 - T - 1), min(nl, k1 + T + 1)
        base = int(Pl[:wa].sum())
        win = oracle.extract(run["ovol"], wa, wb, point_base=base)
        lay = win.voxel_idx[:, 2]
        frozen = (((lay == wa) & (wa > 0)) | ((lay == wb - 1) & (wb < nl))).astype(np.uint8)
        ref = oracle.smooth(win, run["sp"], T, run["lam"], run["d"], frozen=frozen)
        sel = (lay >= k0) & (lay < k1)
        g0 = int(Pl[:k0].sum())
        n = int(sel.sum())
        gpu = pipe.out[g0:g0 + n].cpu().numpy().astype(np.float64)
        err = np.abs(gpu - ref[sel]) / np.array(run["sp"])
        return float(err.max()) if n else 0.0, n

    res = pmap(work, starts)
    assert sum(n for _, n in res) > 0
    worst = max(e for e, _ in res)
    assert worst <= TOL, res


@pytest.mark.parametrize("n", [1, 8, 64])
def test_c6_label_subsets(n):
    """NEXT-1: extracting only labels {1..n} of the Synthetic-like c6 volume
    (general label set: bitset-classified kernels) reproduces the oracle's per-layer counts, and
    a sampled window bit for bit."""
    spec = psn_gen.config("c6")
    p = gu.psn()
    labels = psn_gen.generate_device(spec)
    vol = p.volume(labels)
    ls = list(range(1, n + 1))
    mesh = p.extract(vol, ls)
    host = labels.cpu().numpy()
    ovol = oracle.Volume(host, (spec.M, spec.N, spec.O), 0, (1.0, 1.0, 1.0), label_set=tuple(ls))
    Pl, Ql, Sl = layer_counts_parallel(ovol)
    assert (mesh.n_points, mesh.n_quads, mesh.n_stencil) == (int(Pl.sum()), int(Ql.sum()), int(Sl.sum()))
    k0, k1 = 240, 243
    om = oracle.extract(ovol, k0, k1, point_base=int(Pl[:k0].sum()), stencil_base=int(Sl[:k0].sum()))
    g = gu.mesh_np(mesh)
    p0, s0, q0 = int(Pl[:k0].sum()), int(Sl[:k0].sum()), int(Ql[:k0].sum())
    np.testing.assert_array_equal(g["points"][p0:p0 + om.n_points], om.points)
    np.testing.assert_array_equal(g["quads"][q0:q0 + om.n_quads], om.quads)
    np.testing.assert_array_equal(g["pairs"][q0:q0 + om.n_quads], om.pairs)
    np.testing.assert_array_equal(g["csr_ids"][s0:s0 + om.n_stencil], om.csr_ids)
