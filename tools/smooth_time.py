"""Time psn_smooth alone (whole volume, per-iteration schedule, the bench's launch configuration) and
print a digest of the smoothed coordinates, so library builds can be compared (PSN_LIB selects the
build; tools/ab.py builds them).  GPU only.

    for l in base new; do PSN_LIB=ab/libpsn_$l.so python tools/smooth_time.py --config c4; done
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import psn_gen  # noqa: E402
from paper_2401_14906_b200.psn import PSN, Pipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--graph", action="store_true", help="replay psn_smooth captured in a CUDA graph (as bench.py)")
    a = ap.parse_args()
    spec = psn_gen.config(a.config)
    T, lam, d = psn_gen.SMOOTHING[a.config]
    p = PSN(0)
    vol = p.volume(psn_gen.generate_device(spec), spacing=tuple(spec.spacing))
    pipe = Pipeline(p, vol, T, lam, d)
    pipe.run()
    for _ in range(2):
        pipe.smooth()
    run = pipe.smooth
    if a.graph:
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            pipe.smooth()
        run = g.replay
        run()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(a.reps):
        run()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.reps
    P = pipe.counts[0]
    x = pipe.out[:P].contiguous().view(torch.int32).to(torch.int64)
    dig = int((x * torch.arange(1, x.numel() + 1, device=x.device).view(x.shape)).sum()) % (1 << 61)
    print(json.dumps({"config": a.config, "lib": os.path.basename(os.environ.get("PSN_LIB", "default")), "P": P,
                      "T": T, "graph": a.graph, "smooth_ms": ms, "per_iter_us": 1e3 * ms / T, "digest": dig}), flush=True)


if __name__ == "__main__":
    main()
