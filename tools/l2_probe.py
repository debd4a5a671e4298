"""Probe: how much faster are counting / emission when a z-slab's labels are
L2-resident (i.e. would a z-chunked count -> emit schedule pay)?  GPU only.

    python tools/l2_probe.py --config c4 --layers 24 48 96
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import psn_gen  # noqa: E402
from paper_2401_14906_b200.psn import PSN  # noqa: E402


def timed(fn):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--layers", type=int, nargs="*", default=[24, 48, 96])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--async", dest="asyn", action="store_true",
                    help="only run flush + PSN_COUNT|PSN_EMIT per rep (for an ncu launch list with --cache-control "
                         "none vs all: the emission kernel's duration with / without the slab's labels in L2)")
    a = ap.parse_args()
    spec = psn_gen.config(a.config)
    p = PSN(0)
    full = psn_gen.generate_device(spec)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    O = full.shape[0]
    for L in a.layers + [O]:
        k0 = (O - L) // 2
        lab = full[k0:k0 + L]
        vol = p.volume(lab, spacing=tuple(spec.spacing))
        labels = p.labels(None)
        ws = p.workspace(vol)
        counted = p.count(vol, labels, ws)
        mesh = p.emit(vol, labels, ws, counted)
        res = {"layers": L, "points": counted.n_points}
        if a.asyn:
            for _ in range(a.reps):
                flush.zero_()
                p.extract_into(vol, labels, ws, mesh)
            torch.cuda.synchronize()
            print(json.dumps(res), flush=True)
            del mesh, ws
            continue
        cold_c, cold_e, hot_e, hot_c = [], [], [], []
        for _ in range(a.reps):
            flush.zero_()
            cold_c.append(timed(lambda: p.count(vol, labels, ws)))
            hot_e.append(timed(lambda: p.emit(vol, labels, ws, counted, mesh=mesh)))
            hot_c.append(timed(lambda: p.count(vol, labels, ws)))
            flush.zero_()
            cold_e.append(timed(lambda: p.emit(vol, labels, ws, counted, mesh=mesh)))
        for k, v in (("count_cold", cold_c), ("count_hot", hot_c), ("emit_hot", hot_e), ("emit_cold", cold_e)):
            v.sort()
            res[k + "_us"] = round(v[len(v) // 2] * 1000, 1)
            res[k + "_us_per_layer"] = round(v[len(v) // 2] * 1000 / (L - 1), 3)
        print(json.dumps(res), flush=True)
        del mesh, ws


if __name__ == "__main__":
    main()
