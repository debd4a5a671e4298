"""Full-size parity at BASELINE.json's configs (c3, c4, c5a, c5b) and the NEXT-1 config c6, in the launch
configuration bench.py times (psn.Pipeline: PSN_COUNT|PSN_EMIT with
preallocated capacities, then psn_smooth).

The oracle is too slow to extract a 1024^3 volume whole in a test, so:
  * totals P, Q, S: oracle per-layer counts over the WHOLE volume (disjoint
    layer ranges evaluated in parallel threads -- the same plain oracle code);
  * sampled layer windows: oracle extraction of layers [k0, k1) with global
    ids, compared bit for bit with the matching slices of the GPU arrays;
  * smoothing: the oracle smooths the window extended by T+1 frozen layers on
    each side (errors from a frozen layer travel one stencil hop per
    iteration, so the inner layers are exact -- pinned on CPU by
    test_window_smoothing_matches_full); GPU within 1e-4 x spacing.
"""
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


def layer_counts_parallel(vol, nthreads=8):
    O = vol.dims[2]
    nl = O - 1
    bounds = [(i * nl // nthreads, (i + 1) * nl // nthreads) for i in range(nthreads)]
    with ThreadPoolExecutor(nthreads) as ex:
        parts = list(ex.map(lambda b: oracle.layer_counts(vol, b[0], b[1]), bounds))
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
    host = labels.cpu().numpy()
    ovol = oracle.Volume(host, (spec.M, spec.N, spec.O), 0, sp)
    Pl, Ql, Sl = layer_counts_parallel(ovol)
    yield dict(name=name, spec=spec, pipe=pipe, host=host, ovol=ovol, Pl=Pl, Ql=Ql, Sl=Sl, T=T, lam=lam, d=d, sp=sp)
    del pipe, labels
    torch.cuda.empty_cache()


def test_totals(run):
    pipe = run["pipe"]
    assert pipe.counts == (int(run["Pl"].sum()), int(run["Ql"].sum()), int(run["Sl"].sum()))


def _windows(O, n=3, width=3):
    nl = O - 1
    ks = [1, nl // 2 - width // 2, nl - width - 1]
    return [(max(0, k), min(nl, k + width)) for k in ks[:n]]


def test_sampled_windows_bit_exact(run):
    pipe, Pl, Ql, Sl = run["pipe"], run["Pl"], run["Ql"], run["Sl"]
    spec = run["spec"]
    m = pipe.mesh
    for k0, k1 in _windows(spec.O):
        pb, qb, sb = int(Pl[:k0].sum()), int(Ql[:k0].sum()), int(Sl[:k0].sum())
        om = oracle.extract(run["ovol"], k0, k1, point_base=pb, stencil_base=sb)
        P, Q = om.n_points, om.n_quads
        np.testing.assert_array_equal(m.points[pb:pb + P].cpu().numpy(), om.points)
        np.testing.assert_array_equal(m.quads[qb:qb + Q].cpu().numpy().view(np.uint32), om.quads)
        np.testing.assert_array_equal(m.pairs[qb:qb + Q].cpu().numpy().view(np.uint32), om.pairs)
        np.testing.assert_array_equal(m.stencil_offsets[pb:pb + P + 1].cpu().numpy().view(np.uint32), om.csr_off)
        np.testing.assert_array_equal(m.stencil_ids[sb:sb + om.n_stencil].cpu().numpy().view(np.uint32), om.csr_ids)
        np.testing.assert_array_equal(m.face_masks[pb:pb + P].cpu().numpy(), om.face_mask)


def test_sampled_smoothing(run):
    pipe, Pl = run["pipe"], run["Pl"]
    spec, T = run["spec"], run["T"]
    nl = spec.O - 1
    k0 = nl // 2 - 1
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
    assert err.max() <= TOL, err.max()


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
