"""Time psn_smooth alone (whole volume, bench launch config) for the smoothing
strategies: per-iteration vs wavefront over (G, tile).  GPU only.

    python tools/tb_sweep.py --config c4 --G 5 10 20 --tile 512 1024 2048
"""
import argparse
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import psn_gen  # noqa: E402
from paper_2401_14906_b200.psn import PSN, Pipeline  # noqa: E402


def timeit(fn, reps):
    for _ in range(2):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--G", type=int, nargs="*", default=[0])
    ap.add_argument("--tile", type=int, nargs="*", default=[0])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    spec = psn_gen.config(a.config)
    T, lam, d = psn_gen.SMOOTHING[a.config]
    p = PSN(0)
    labels = psn_gen.generate_device(spec)
    vol = p.volume(labels, spacing=tuple(spec.spacing))
    pipe = Pipeline(p, vol, T, lam, d)
    pipe.run()
    p.set_smoothing(1, 0)
    ms = timeit(pipe.smooth, a.reps)
    ref = pipe.out.clone()
    res = {"config": a.config, "P": pipe.counts[0], "T": T, "per_iteration_ms": ms, "wavefront": []}
    print(f"{a.config} P={pipe.counts[0]} per-iteration {ms:.3f} ms", flush=True)
    for G, tile in itertools.product(a.G, a.tile):
        p.set_smoothing(0, G, tile)
        ms = timeit(pipe.smooth, a.reps)
        p.smooth_status(pipe.mesh, pipe.sws)
        same = bool(torch.equal(pipe.out, ref))
        res["wavefront"].append({"G": G, "tile": tile, "ms": ms, "bit_identical": same})
        print(f"  wavefront G={G} tile={tile}: {ms:.3f} ms identical={same}", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
