"""NEXT-1 (Fig. "Relative slowdown as the number of labels
increases"): time extraction (+ smoothing) of the Synthetic-like c6 volume
while extracting only labels {1..n}, n = 1 .. 128, through the general
(bitset-classified) label path; all_nonzero for reference.  GPU only.

    python tools/label_sweep.py [--config c6] [--reps 5]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import psn_gen  # noqa: E402
from paper_2401_14906_b200.psn import PSN, Pipeline  # noqa: E402


def timed(fn, reps, flush):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c6")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    spec = psn_gen.config(a.config)
    T, lam, d = psn_gen.SMOOTHING[a.config]
    p = PSN(0)
    labels = psn_gen.generate_device(spec)
    vol = p.volume(labels, spacing=tuple(spec.spacing))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for n in [1, 2, 4, 8, 16, 32, 64, 128, None]:
        ls = None if n is None else list(range(1, n + 1))
        pipe = Pipeline(p, vol, T, lam, d, label_set=ls)
        t_ext = timed(pipe.extract, a.reps, flush)
        t_sm = timed(pipe.smooth, a.reps, flush)
        rows.append({"labels": "all_nonzero" if n is None else n, "points": pipe.counts[0], "quads": pipe.counts[1],
                     "extract_ms": t_ext, "smooth_ms": t_sm, "total_ms": t_ext + t_sm})
        print(json.dumps(rows[-1]), flush=True)
        del pipe
        torch.cuda.empty_cache()
    base = rows[0]["total_ms"]
    for r in rows:
        r["relative_slowdown"] = r["total_ms"] / base
    print(json.dumps({"config": a.config, "T": T, "sweep": rows}))


if __name__ == "__main__":
    main()
