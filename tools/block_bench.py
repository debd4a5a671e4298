"""Time the NEXT-4 block path (psn_block_gather -> psn_extract -> psn_stitch_*) against the
whole-volume extraction on a BASELINE config (CUDA events around each whole run, after warm-up).

    python tools/block_bench.py --config c4 --blocks 2,2,2 --reps 3

Prints one JSON line per variant: whole (device labels, psn.extract); blocks in-core (device labels,
local meshes kept); blocks from pinned host labels (one label box resident at a time, local meshes
kept); the same with only one block resident at all (re-gathered and re-extracted in the emit pass).  Each run includes its host synchronisations (the COUNT read-backs, the stitch totals).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import psn_gen  # noqa: E402
from paper_2401_14906_b200 import PSN  # noqa: E402
from paper_2401_14906_b200.blocks import BlockedExtractor  # noqa: E402


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        del out
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--blocks", default="2,2,2")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    blocks = tuple(int(x) for x in args.blocks.split(","))
    spec = psn_gen.config(args.config)
    M, N, O = (int(d) for d in spec.dims)
    sp = tuple(float(s) for s in spec.spacing)
    dev = psn_gen.generate_device(spec)
    host = dev.cpu().pin_memory()
    p = PSN(0)
    vol = p.volume(dev, spacing=sp)
    ws = p.workspace(vol)
    p.extract(vol, ws=ws)   # warm-up
    vox = (M - 1) * (N - 1) * (O - 1)
    rows = []
    t = timed(lambda: p.extract(vol, ws=ws), args.reps)
    rows.append({"variant": "whole", "ms": t})
    bx = BlockedExtractor(p, (M, N, O), blocks=blocks, spacing=sp, keep_local=True)
    bx.run(dev)
    rows.append({"variant": "blocks_in_core", "ms": timed(lambda: bx.run(dev), args.reps)})
    bh = BlockedExtractor(p, (M, N, O), blocks=blocks, spacing=sp, keep_local=True)
    bh.run(host)
    rows.append({"variant": "blocks_host_labels", "ms": timed(lambda: bh.run(host), args.reps)})
    bo = BlockedExtractor(p, (M, N, O), blocks=blocks, spacing=sp, keep_local=False)
    bo.run(host)
    rows.append({"variant": "blocks_host_labels_one_resident", "ms": timed(lambda: bo.run(host), args.reps)})
    for b_, name, src in ((bx, "blocks_in_core", dev), (bh, "blocks_host_labels", host),
                          (bo, "blocks_host_labels_one_resident", host)):
        b_.timings = {}
        b_.run(src)
        rows.append({"variant": name + "_phases", "ms_by_phase": dict(b_.timings)})
    for r in rows:
        r.update({"config": args.config, "blocks": list(blocks),
                  "label_bytes": int(host.numel() * host.element_size())})
        if "ms" in r:
            r["voxels_per_s"] = vox / (r["ms"] * 1e-3)
        print(json.dumps(r))


if __name__ == "__main__":
    main()
