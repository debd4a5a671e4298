"""Multi-GPU data path emulated on ONE GPU.

Each z-slab is extracted through psn_extract with its one-slice halos, the
cross-rank all-gather is replaced by a host prefix sum, and the smoothing halo
exchange by device copies between the slabs' window buffers.  The rank-order
concatenation must equal the single-GPU output bit for bit (extraction) and
the smoothed coordinates must equal the single-GPU smoothing bit for bit (the
per-point arithmetic is identical), and match the oracle within 1e-4 * s."""
import numpy as np
import pytest
import torch

import gpu_util as gu
import oracle
import psn_gen
from paper_2401_14906_b200.dist import halo_plan, partition, slab_slices

pytestmark = pytest.mark.gpu


def run_slabs(labels_np, G, T=6, lam=0.5, d=0.5, spacing=(1.0, 1.0, 1.0)):
    p = gu.psn()
    O, N, M = labels_np.shape
    parts = partition(O - 1, G)
    vols, wss, counted, devs = [], [], [], []
    for (k0, k1) in parts:
        z_lo, z_hi = slab_slices(O, k0, k1)
        dev = torch.from_numpy(np.ascontiguousarray(labels_np[z_lo:z_hi])).cuda()
        vol = p.volume(dev, dims=(M, N, O), spacing=spacing, z_lo=z_lo, own=(k0, k1))
        ws = p.workspace(vol)
        c = p.count(vol, p.labels(None), ws)
        vols.append(vol); wss.append(ws); counted.append(c); devs.append(dev)
    table = torch.tensor([[c.n_points, c.n_quads, c.n_stencil, c.halo_lo_points, c.halo_hi_points] for c in counted])
    meshes = []
    for r in range(G):
        first = tuple(int(x) for x in table[:r, :3].sum(0)) if r else (0, 0, 0)
        meshes.append(p.emit(vols[r], p.labels(None), wss[r], counted[r], first=first))
    # smoothing with emulated halo exchange
    bufs = [[p.offsets_buffer(m.n_window, "cuda") for _ in range(2)] for m in meshes]   # float4 offsets
    sws = [p.smooth_workspace(m) for m in meshes]
    for r in range(G):
        p.smooth_prepare(vols[r], meshes[r], sws[r])
    plans = [halo_plan(table, r) for r in range(G)]
    src = [None] * G
    for t in range(T):
        for r in range(G):
            p.smooth_step(vols[r], meshes[r], sws[r], src[r], bufs[r][t & 1], lam, d)
        for r in range(G):   # exchange: r's first layer -> r-1's upper halo, r's last layer -> r+1's lower halo
            dst = bufs[r][t & 1]
            if plans[r]["send_lo"] is not None:
                a, b = plans[r]["send_lo"]; c_, d_ = plans[r - 1]["recv_hi"]
                bufs[r - 1][t & 1][c_:d_] = dst[a:b]
            if plans[r]["send_hi"] is not None:
                a, b = plans[r]["send_hi"]; c_, d_ = plans[r + 1]["recv_lo"]
                bufs[r + 1][t & 1][c_:d_] = dst[a:b]
        src = [bufs[r][t & 1] for r in range(G)]
    outs = []
    for r in range(G):
        out = torch.empty((max(meshes[r].n_window, 1), 3), dtype=torch.float32, device="cuda")
        p.smooth_finalize(vols[r], meshes[r], src[r], out)
        outs.append(out)
    torch.cuda.synchronize()
    return meshes, outs, table


def concat(meshes, outs):
    g = {k: [] for k in ("points", "quads", "pairs", "csr_ids", "face_mask", "smoothed")}
    offs = []
    for m, o in zip(meshes, outs):
        d = gu.mesh_np(m)
        hl, P = m.c.halo_lo_points, m.n_points
        g["points"].append(d["points"][hl:hl + P])
        g["smoothed"].append(o[hl:hl + P].cpu().numpy())
        for k in ("quads", "pairs", "csr_ids", "face_mask"):
            g[k].append(d[k])
        offs.append(d["csr_off"][:-1])
        last = d["csr_off"][-1:]
    out = {k: np.concatenate(v) for k, v in g.items()}
    out["csr_off"] = np.concatenate(offs + [last])
    return out


@pytest.mark.parametrize("G", [2, 3, 5])
def test_slab_emulation_matches_single(G):
    rng = np.random.default_rng(100 + G)
    a = np.zeros((23, 21, 37), np.uint16)
    a[1:-1, 1:-1, 1:-1] = rng.integers(0, 4, size=(21, 19, 35))
    z, y, x = np.meshgrid(np.arange(23), np.arange(21), np.arange(37), indexing="ij")
    a[((x - 18) ** 2 + (y - 10) ** 2 + (z - 11) ** 2) < 30] = 9
    T = 6
    meshes, outs, table = run_slabs(a, G, T)
    g = concat(meshes, outs)
    p, vol, m1, _ = gu.gpu_extract(a)
    single = gu.mesh_np(m1)
    for k in ("points", "quads", "pairs", "csr_off", "csr_ids", "face_mask"):
        np.testing.assert_array_equal(g[k], single[k], err_msg=k)
    s1 = p.smooth(vol, m1, T, 0.5, 0.5)
    np.testing.assert_array_equal(g["smoothed"], s1[:m1.n_points].cpu().numpy())
    om = oracle.extract(oracle.as_volume(a))
    ref = oracle.smooth(om, (1, 1, 1), T, 0.5, 0.5)
    assert np.abs(g["smoothed"].astype(np.float64) - ref).max() <= 1e-4


def test_slab_emulation_c2_four_slabs():
    spec = psn_gen.config("c2")
    host = psn_gen.generate_host(spec)
    meshes, outs, _ = run_slabs(host, 4, T=25)
    g = concat(meshes, outs)
    om = oracle.extract(oracle.as_volume(host))
    gu.assert_mesh_equal({k: g[k] for k in ("points", "quads", "pairs", "csr_off", "csr_ids", "face_mask")}, om)
    ref = oracle.smooth(om, (1, 1, 1), 25, 0.5, 0.5)
    assert np.abs(g["smoothed"].astype(np.float64) - ref).max() <= 1e-4


@pytest.mark.parametrize("G", [2, 3])
def test_device_c1_matches_host_path(G):
    """The multi-GPU steady state without host round trips: PSN_COUNT|PSN_DEVICE ->
    psn_extract_totals -> (all-gather, here a concatenation) + prefix sum on the device ->
    PSN_EMIT|PSN_DEVICE with mesh.first_dev writes exactly what the host-synchronised path writes."""
    from test_gpu_balance import extract_slabs
    p = gu.psn()
    rng = np.random.default_rng(7 + G)
    a = np.zeros((19, 17, 29), np.uint16)
    a[1:-1, 1:-1, 1:-1] = rng.integers(0, 4, size=(17, 15, 27))
    vols, meshes, firsts, total = extract_slabs(p, a, G, (1.0, 1.0, 1.0))
    ref = [gu.mesh_np(m) for m in meshes]
    lab = p.labels(None)
    wss = [p.workspace(v) for v in vols]
    tots = [torch.zeros(5, dtype=torch.int64, device="cuda") for _ in range(G)]
    for r in range(G):
        p.count_device(vols[r], lab, wss[r], tots[r])
    allt = torch.stack(tots)                        # what the NCCL all-gather would deliver
    for r in range(G):
        m = meshes[r]
        for t in (m.points, m.quads, m.pairs, m.stencil_offsets, m.stencil_ids, m.face_masks):
            t.zero_()
        first = allt[:r, :3].sum(0)
        p.emit_device(vols[r], lab, wss[r], m, first)
    torch.cuda.synchronize()
    for r in range(G):
        got = gu.mesh_np(meshes[r])
        for k in ref[r]:
            np.testing.assert_array_equal(got[k], ref[r][k])
        assert tuple(int(x) for x in tots[r].tolist()) == (meshes[r].n_points, meshes[r].n_quads, meshes[r].n_stencil,
                                                            meshes[r].c.halo_lo_points, meshes[r].c.halo_hi_points)
