"""Time psn_extract (PSN_COUNT|PSN_EMIT, steady state) alone on a config's
volume, with an L2 flush before every run; optional count check.  GPU only.

    python tools/ext_time.py --config c4 --reps 10
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
    ap.add_argument("--warmup", type=int, default=3)
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
    times = []
    for _ in range(a.reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        pipe.extract()
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    ok = pipe.check()
    times.sort()
    print(json.dumps({"config": a.config, "counts": pipe.counts, "counts_ok": ok,
                      "ms_min": times[0], "ms_med": times[len(times) // 2],
                      "ms_mean": sum(times) / len(times)}))


if __name__ == "__main__":
    main()
