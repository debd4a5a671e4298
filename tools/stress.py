"""Randomised parity stress run (GPU): random shapes (odd / even / 16-byte-multiple row widths),
dtypes, label sets, spacings and block grids; every case must match the oracle bit for bit (extraction)
or within the smoothing tolerance, and the stitched blocks must equal the whole-volume mesh.

    python tools/stress.py --seconds 240 --seed 1
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import gpu_util as gu  # noqa: E402
from paper_2401_14906_b200.blocks import BlockedExtractor  # noqa: E402


def volume(rng):
    dtype = rng.choice([np.uint8, np.uint16, np.uint32])
    M = int(rng.choice([2, 3, int(rng.integers(4, 80)), int(rng.integers(80, 700))]))
    N = int(rng.integers(2, 40)); O = int(rng.integers(2, 30))
    if M * N * O > 2_000_000:
        O = max(2, 2_000_000 // (M * N))
    kind = rng.integers(0, 3)
    if kind == 0:
        a = rng.integers(0, int(rng.integers(2, 6)), (O, N, M))
    else:
        z, y, x = np.meshgrid(np.arange(O), np.arange(N), np.arange(M), indexing="ij")
        a = np.zeros((O, N, M), np.int64)
        for lab in range(1, int(rng.integers(2, 9))):
            c = rng.uniform(0, 1, 3) * np.array([M, N, O])
            r = rng.uniform(1.5, max(1.6, 0.6 * max(M, N, O)))
            a[(x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 <= r * r] = lab
        if kind == 2:
            m = rng.random(a.shape) < 0.05
            a[m] = rng.integers(0, 9, int(m.sum()))
    a = a.astype(dtype)
    if dtype == np.uint32:
        a = (a.astype(np.uint64) * 2654435761 % (1 << 32)).astype(np.uint32)
    vals = np.unique(a)
    ls = None
    if rng.random() < 0.4 and len(vals) > 1:
        pick = vals[rng.random(len(vals)) < 0.5]
        ls = [int(v) for v in pick] or [int(vals[-1])]
    sp = tuple(float(s) for s in rng.choice([0.5, 0.8, 1.0, 1.5], 3))
    org = tuple(float(o) for o in rng.uniform(-10, 10, 3))
    return a, ls, sp, org


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=240)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    p = gu.psn()
    t0 = time.time()
    n = 0
    while time.time() - t0 < args.seconds:
        a, ls, sp, org = volume(rng)
        O, N, M = a.shape
        ctx = f"case {n}: shape {a.shape} {a.dtype} ls={None if ls is None else len(ls)} sp={sp}"
        _, vol, mesh, dev = gu.gpu_extract(a, sp, org, ls)
        om = oracle.extract(oracle.as_volume(a, sp, org, ls))
        try:
            assert (mesh.n_points, mesh.n_quads, mesh.n_stencil) == (om.n_points, om.n_quads, om.n_stencil)
            gu.assert_mesh_equal(gu.mesh_np(mesh), om)
            if om.n_points:
                T = int(rng.integers(1, 8))
                pts = p.smooth(vol, mesh, T, 0.5, 0.5)[:om.n_points].cpu().numpy().astype(np.float64)
                ref = oracle.smooth(om, sp, T, 0.5, 0.5)
                half_ulp = 0.5 * np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
                err = ((np.abs(pts - ref) - half_ulp) / np.array(sp)).max()
                assert err <= 1e-4, f"smoothing err {err}"
            blocks = tuple(int(rng.integers(1, 4)) for _ in range(3))
            ms = BlockedExtractor(p, (M, N, O), blocks=blocks, spacing=sp, origin=org, label_set=ls,
                                  keep_local=bool(rng.random() < 0.5)).run(dev)
            g, w = gu.mesh_np(ms), gu.mesh_np(mesh)
            for k in g:
                np.testing.assert_array_equal(g[k], w[k], err_msg=f"blocks {blocks} {k}")
        except AssertionError as e:
            print("FAIL", ctx, e, flush=True)
            np.save(f"gpurun_out/stress_fail_{n}.npy", a)
            raise
        n += 1
    print(f"stress ok: {n} cases in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
