"""Per-pass times of psn_extract (PSN_COUNT|PSN_EMIT, steady state) on a config's volume:
count (incl. header reset), scan, emission -- events recorded by the library between its
launches (psn_ctx_set_pass_events); L2 flushed before every run.  GPU only.  PSN_LIB selects
the library build (A/B runs: tools/ab.py).

    python tools/pass_time.py --config c4 --reps 20
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import psn_gen  # noqa: E402
from paper_2401_14906_b200.psn import PSN, Pipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--digest", action="store_true", help="also print a digest of the outputs")
    a = ap.parse_args()
    spec = psn_gen.config(a.config)
    T, lam, d = psn_gen.SMOOTHING[a.config]
    p = PSN(0)
    labels = psn_gen.generate_device(spec)
    vol = p.volume(labels, spacing=tuple(spec.spacing))
    pipe = Pipeline(p, vol, T, lam, d)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(a.warmup):
        pipe.extract()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(a.reps)]
    for r in range(a.reps):
        flush.zero_()
        p.set_pass_events(evs[r])
        pipe.extract()
    torch.cuda.synchronize()
    p.set_pass_events(None)
    per = [[e[i].elapsed_time(e[i + 1]) for e in evs] for i in range(3)]
    tot = [e[0].elapsed_time(e[3]) for e in evs]
    out = {"config": a.config, "lib": os.environ.get("PSN_LIB", "default"), "counts": pipe.counts,
           "count_ms": statistics.median(per[0]), "scan_ms": statistics.median(per[1]),
           "emit_ms": statistics.median(per[2]), "total_ms": statistics.median(tot)}
    if a.digest:
        m = pipe.mesh
        P, Q, S = pipe.counts
        h = 0
        for t in (m.points[:P], m.quads[:Q], m.pairs[:Q], m.stencil_offsets[:P + 1], m.stencil_ids[:S],
                  m.face_masks[:P]):
            x = t.contiguous().view(torch.int32 if t.dtype != torch.uint8 else torch.uint8).to(torch.int64)
            h = (h * 1000003 + int((x * torch.arange(1, x.numel() + 1, device=x.device).view(x.shape)).sum())) % (1 << 61)
        out["digest"] = h
        out["ok"] = pipe.check()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
