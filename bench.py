#!/usr/bin/env python
"""bench.py -- PSN hot path on B200: extraction (k_count3 -> k_scan -> k_emit_band) +
T-iteration constrained smoothing (k_smooth_prep8 + T x k_smooth_v4), timed with CUDA events.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl psn|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL): the c4 volume is
z-slab partitioned (strong scaling, total work fixed), with the all-gather of
per-rank totals (C1), the point-balanced re-cut of the smoothing (C4) and the
per-iteration halo exchange (C2), fused into the smoothing kernel as NVLink
peer pushes (--nccl-halo: NCCL point-to-point instead).

One JSON line on rank 0.  `value` = label voxels of the whole volume pushed
through one step (extraction + T smoothing iterations) per second; the
`extract` / `smooth` sub-objects give the two halves of BASELINE.json's metric
(voxels/s extracted, smoothed point-iterations/s) and their HBM roofline
fractions.  `--impl reference` times the oracle (oracle/, plain C, 1 core) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "label voxels/s extracted + smoothed point-iters/s, % of HBM roofline, 1–8 GPU"
WORKLOADS = {
    "c1": "c1: 32^3 u16, 3 spheres; extract + 10 smoothing iterations (lambda 0.5, box 0.5 voxel)",
    "c2": "c2: 256^3 u8, 20-seed Voronoi in an ellipsoid; extract + 25 smoothing iterations + shortest-diagonal triangulation",
    "c3": "c3: 512x512x600 u16 torso-like, spacing 0.8x0.8x1.5, 101 labels; extract + 25 smoothing iterations",
    "c4": "c4: 1024^3 u16 atlas-like (200 Voronoi labels in a ball + 300 inclusions); extract + 50 smoothing iterations, z-slab over N GPUs",
    "c5a": "c5a: 512^3 u8 iid {0,1,2,3}; extract + 10 smoothing iterations",
    "c5b": "c5b: 512^3 u8 single sphere r=16; extract + 10 smoothing iterations",
    "c6": "c6 (NEXT-1): 512^3 u16 Synthetic-like, 128 overlapping spheres (P 5.22 M, Q 5.25 M); extract + 25 smoothing iterations",
}
TRIANGULATE = {"c2"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def profile_traffic(kernel: str, config: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d[config][kernel]
        return float(e["dram_bytes_per_launch"])
    except Exception:
        return None


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, start: bool):
        """Bracket the timed region (samples outside it are dropped, nearest kept if none)."""
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons, util = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", 0.0), getattr(self, "t1", 1e300)
        inside = [ln for ts, ln in self.lines if t0 <= ts <= t1 + 0.05]
        if not inside and self.lines:   # region shorter than the sampling period: nearest samples
            inside = [ln for ts, ln in sorted(self.lines, key=lambda x: abs(x[0] - 0.5 * (t0 + t1)))[:2]]
        for ln in inside:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0])); mx.append(float(f[1])); util.append(float(f[6]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [s for s, u in zip(sm, util) if u > 0] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- byte model
def algorithmic_bytes(V, b, P, Q, S):
    """B_ext = V*b + 12P + 16Q + 8Q + 4(P+1) + 4S; B_sm/iter = 24P + 4(P+1) + 4S."""
    b_ext = V * b + 12 * P + 24 * Q + 4 * (P + 1) + 4 * S
    b_sm = 24 * P + 4 * (P + 1) + 4 * S
    return b_ext, b_sm


# --------------------------------------------------------------------------- oracle (CPU baseline / reference arm)
def sample_window(O: int, n_layers: int):
    """Central voxel layers [k0, k1) plus one frozen layer each side [wa, wb) and
    the lattice slices [z_lo, z_hi) the oracle needs for them."""
    n_layers = max(1, min(n_layers, O - 1))
    k0 = max(0, min((O - 1) // 2 - n_layers // 2, O - 1 - n_layers))
    k1 = k0 + n_layers
    wa, wb = max(k0 - 1, 0), min(k1 + 1, O - 1)
    z_lo, z_hi = max(wa - 1, 0), min(wb + 1, O - 1) + 1
    return n_layers, k0, k1, wa, wb, z_lo, z_hi


def oracle_sample(cfg: str, n_layers: int, labels_host=None):
    """Time the oracle (plain C, single thread) on voxel layers [k0, k0+n_layers) of the
    config: extraction + T fp64 smoothing iterations.  The extracted window carries one
    frozen voxel layer on each interior side so every stencil id stays inside it.
    Returns (seconds, voxels, (k0, k1), labels_host)."""
    import numpy as np

    import oracle
    import psn_gen
    spec = psn_gen.config(cfg)
    M, N, O = spec.M, spec.N, spec.O
    T, lam, d = psn_gen.SMOOTHING[cfg]
    n_layers, k0, k1, wa, wb, z_lo, z_hi = sample_window(O, n_layers)
    if callable(labels_host):
        labels_host = labels_host(z_lo, z_hi)
    if labels_host is None:
        labels_host = psn_gen.generate_host(spec, z_lo, z_hi)
    vol = oracle.Volume(np.ascontiguousarray(labels_host), (M, N, O), z_lo, tuple(spec.spacing))
    with pinned_core0():
        t0 = time.perf_counter()
        mesh = oracle.extract(vol, wa, wb)
        lay = mesh.voxel_idx[:, 2]
        frozen = (((lay == wa) & (wa < k0)) | ((lay == wb - 1) & (wb > k1))).astype(np.uint8)
        oracle.smooth(mesh, tuple(spec.spacing), T, lam, d, frozen=frozen)
        dt = time.perf_counter() - t0
    return dt, M * N * n_layers, (k0, k1), labels_host


_PINNED = {"core": None}


def host_info():
    """lscpu model, online CPUs, and the core the oracle was pinned to (SURVEY 8(d) oracle timing;
    None if the pinning was refused, e.g. core 0 outside the process's cpuset)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.strip().lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "pinned_core": _PINNED["core"], "threads_used": 1}


class pinned_core0:
    """Run the (single-threaded) oracle pinned to core 0 (taskset -c 0 equivalent for this thread)."""

    def __enter__(self):
        try:
            self.old = os.sched_getaffinity(0)
            os.sched_setaffinity(0, {0})
            _PINNED["core"] = 0
        except Exception:
            self.old = None
            _PINNED["core"] = None
        return self

    def __exit__(self, *exc):
        if self.old is not None:
            try:
                os.sched_setaffinity(0, self.old)
            except Exception:
                pass


# --------------------------------------------------------------------------- reference arm
def sample_text(cfg, k0, k1, vox, T, reps=None):
    r = f", repeated {reps}x" if reps else ""
    return (f"{cfg} voxel layers [{k0},{k1}) ({vox} voxels){r}: oracle extract + {T}-iteration fp64 smoothing, "
            f"single thread pinned to core 0 (the same window the reference arm times per step)")


def sample_layers(cfg, voxels):
    import psn_gen
    spec = psn_gen.config(cfg)
    return max(1, int(round(voxels / (spec.M * spec.N))))


def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    cfg = args.config
    import psn_gen
    spec = psn_gen.config(cfg)
    # bounded sample per step (~1-2 s of single-core oracle work): the same window cpu_baseline times
    n_layers = sample_layers(cfg, args.ref_voxels)
    labels = None
    times = []
    for s in range(args.warmup + args.steps):
        dt, vox, (k0, k1), labels = oracle_sample(cfg, n_layers, labels_host=labels)
        if s >= args.warmup:
            times.append(dt)
    t = sum(times)
    value = vox * len(times) / t
    sample = sample_text(cfg, k0, k1, vox, psn_gen.SMOOTHING[cfg][0])
    line = {"metric": METRIC, "value": value, "unit": "voxel/s", "n_gpus": max(world, args.gpus), "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u16/f64" if spec.elem_bytes == 2 else "u8/f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOADS[cfg], "sample": sample},
            "cpu_baseline": {"value": value, "unit": "voxel/s", "cores": 1, "kind": "oracle", "sample": sample,
                             "host": host_info()},
            "e2e": {"value": value, "unit": "voxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm
def run_psn(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import psn_gen
    from paper_2401_14906_b200 import PSN
    from paper_2401_14906_b200.psn import Pipeline, SurfaceNetsStream, surface_nets_host

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = args.config
    spec = psn_gen.config(cfg)
    M, N, O = spec.M, spec.N, spec.O
    b = spec.elem_bytes
    V = M * N * O
    T, lam, d = psn_gen.SMOOTHING[cfg]
    sp = tuple(spec.spacing)
    psn = PSN(local_rank)
    stream = torch.cuda.current_stream()
    tri = cfg in TRIANGULATE

    if world == 1:
        labels = psn_gen.generate_device(spec)
        vol = psn.volume(labels, spacing=sp)
        pipe = Pipeline(psn, vol, T, lam, d, triangulate=tri, smooth_cache=args.smooth_cache)
        P, Q, S = pipe.counts
        run_extract, run_smooth = pipe.extract, pipe.smooth
        if not args.no_graph:
            # warm the library's one-time host setup, then replay the step as two CUDA graphs (one launch
            # each): the small configs are bound by the per-kernel host launch path otherwise
            pipe.run()
            # the smoothing graph records two events around its T Jacobi launches (psn_ctx_set_smooth_events):
            # k_smooth_v4's mean launch time for the roofline, replayed back to back as in the timed steps
            pipe.capture()
            run_extract, run_smooth = pipe.replay_extract, pipe.replay_smooth
            # one smoothing graph per timed step, each recording its own event pair around the T Jacobi
            # launches: the roofline's launch time is the mean over ALL timed steps (a single step's pair
            # picked up one slow replay in some runs)
            sm_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
            sm_graphs = []
            for e2 in sm_ev:
                psn.set_smooth_events(e2)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    pipe.smooth()
                sm_graphs.append(g)
            psn.set_smooth_events(None)
            torch.cuda.synchronize()
    else:
        from paper_2401_14906_b200.dist import (SlabPipeline, balanced_layer_cuts, gather_layer_points,
                                                partition, slab_slices)
        own = partition(O - 1, world)[rank]

        def make(own_):
            z_lo, z_hi = slab_slices(O, own_[0], own_[1])
            lab_ = psn_gen.generate_device(spec, z_lo, z_hi)
            # C2 fused into the smoothing kernel (peer pushes over NVLink) unless --nccl-halo
            return lab_, SlabPipeline(psn, lab_, (M, N, O), sp, (0.0, 0.0, 0.0), own_, T, lam, d,
                                      peer=not args.nccl_halo)

        labels, pipe = make(own)
        if args.partition == "points":
            # equal z-slabs leave c4's per-rank point counts at up to 1.5x the mean at 8 ranks and
            # smoothing is ~85 % of the step: re-cut the LAYERS once so every rank holds ~P/N points
            # (from the per-layer counts, all-gathered), then extract and smooth on those slabs --
            # no per-step re-partition (C4) or shard assembly
            layer_pts = gather_layer_points(psn, pipe.vol, pipe.ws, own)
            own = balanced_layer_cuts(layer_pts, world)[rank]
            del pipe, labels
            torch.cuda.empty_cache()
            labels, pipe = make(own)
        tab = pipe.table
        P, Q, S = (int(x) for x in tab[:, :3].sum(0))
        run_extract = pipe.extract
        # --partition c4: equal extraction slabs and the point-balanced smoothing re-partition (C4)
        # every step; --partition equal: smoothing on the extraction slabs
        run_smooth = pipe.smooth_balanced if args.partition == "c4" else pipe.smooth
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    clk = ClockSampler(local_rank)
    # warm-up (W >= 3)
    for _ in range(args.warmup):
        run_extract()
        run_smooth()
    torch.cuda.synchronize()
    if world == 1:
        assert pipe.check(), "steady-state totals differ from the warm-up count"
    else:
        pipe.check_totals()
    halo_peer = False
    if world > 1:
        ph = pipe.balanced.peer if args.partition == "c4" else pipe.peer_halo
        halo_peer = ph is not None
    launches = 0
    if world == 1:
        launches = sum(pipe.launches.values())

    K = args.steps
    graphs = world == 1 and not args.no_graph
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    # per-pass events recorded by the library between its launches (psn_ctx_set_pass_events)
    pev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    for e4 in pev:
        for e in e4:
            e.record(stream)
    L2_BYTES = 126e6
    flush = torch.empty(int(2 * L2_BYTES), dtype=torch.uint8, device=dev) if V * b <= L2_BYTES else None
    barrier()
    torch.cuda.synchronize()
    clk.__enter__()
    time.sleep(0.5)          # nvidia-smi needs a moment before its first sample
    barrier()
    torch.cuda.synchronize()
    clk.mark(True)
    for s in range(K):
        if flush is not None:   # inputs fit in L2: flush it between timed steps (outside the events)
            flush.zero_()
        if not graphs:
            psn.set_pass_events(pev[s])
        ev[s][0].record(stream)
        run_extract()
        ev[s][1].record(stream)
        if graphs:
            sm_graphs[s].replay()   # the step's own smoothing graph (same kernels, its own event pair)
        else:
            run_smooth()
        ev[s][2].record(stream)
    torch.cuda.synchronize()
    clk.mark(False)
    psn.set_pass_events(None)
    # Jacobi launch time inside the timed region: every timed step's smoothing graph recorded two events
    # around its T launches; the mean over the K timed steps
    t_v4_live = (sum(e2[0].elapsed_time(e2[1]) for e2 in sm_ev) / len(sm_ev) / T) if (graphs and T > 0) else None
    if graphs:   # per-pass times from K direct (non-graph) extractions: the pass events are host calls
        for s in range(K):
            if flush is not None:
                flush.zero_()
            psn.set_pass_events(pev[s])
            pipe.extract()
        torch.cuda.synchronize()
        psn.set_pass_events(None)
    # k_smooth_v4 launch time (roofline): events around the T Jacobi launches (the one-off cache preparation
    # excluded) -- in graph mode recorded by the captured smoothing graph, K replays after the timed region;
    # else around K direct psn_smooth calls
    t_v4 = t_v4_live
    if world == 1 and T > 0 and t_v4 is None:
        samples = []
        if True:
            sev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
            for s in range(K):
                psn.set_smooth_events(sev[s])
                pipe.smooth()
            torch.cuda.synchronize()
            psn.set_smooth_events(None)
            samples = [e[0].elapsed_time(e[1]) for e in sev]
        t_v4 = sum(samples) / len(samples) / T
    barrier()
    time.sleep(0.05)
    clk.__exit__(None, None, None)
    t_ext = sum(e[0].elapsed_time(e[1]) for e in ev) / K    # ms per step
    t_sm = sum(e[1].elapsed_time(e[2]) for e in ev) / K
    t_step = sum(e[0].elapsed_time(e[2]) for e in ev) / K
    t_pass = [sum(e[i].elapsed_time(e[i + 1]) for e in pev) / K for i in range(3)]   # count, scan, emit
    if world > 1:
        tt = torch.tensor([t_ext, t_sm, t_step, *t_pass], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ext, t_sm, t_step, *t_pass = (float(x) for x in tt.tolist())
    clocks = clk.summary()
    if world > 1 and halo_peer:
        (pipe.balanced.peer if args.partition == "c4" else pipe.peer_halo).check()   # no peer wait timed out

    peak, peak_src = measured_peaks()
    b_ext, b_sm = algorithmic_bytes(V, b, P, Q, S)
    value = V / (t_step * 1e-3)
    ext_vps = V / (t_ext * 1e-3)
    sm_ptit = P * T / (t_sm * 1e-3)
    ext_gbs = b_ext / (t_ext * 1e-3) / 1e9
    # dominant kernel: k_smooth_v4 (T launches per step) -- achieved = B_sm per launch / avg launch time,
    # the launch time taken as (psn_smooth time incl. the one-off k_smooth_prep8) / T (conservative)
    per_launch_ms = t_v4 if t_v4 else t_sm / max(T, 1)
    sm_gbs = b_sm / (t_sm / max(T, 1) * 1e-3) / 1e9          # the smoothing half incl. the cache prep
    v4_gbs = b_sm / (per_launch_ms * 1e-3) / 1e9
    # whole-volume psn_smooth (N = 1) and the peer-push run (N > 1): iterations 2..T are k_smooth_split (split
    # cache); the NCCL-halo steps (--nccl-halo) are k_smooth_v4
    sm_kern = "k_smooth_split" if (T > 1 and (world == 1 or halo_peer)) else "k_smooth_v4"
    dominant = sm_kern if t_sm >= t_ext else "extraction (k_count3+k_scan+k_emit_band)"
    roof = {"bound": "hbm", "kernel": sm_kern, "achieved": v4_gbs / world, "peak": peak, "unit": "GB/s",
            "frac": v4_gbs / world / peak, "traffic": profile_traffic(sm_kern, cfg), "peak_source": peak_src,
            "bytes_per_launch": b_sm / world, "launch_ms": per_launch_ms,
            "note": ("achieved = algorithmic bytes per launch (24P + 4(P+1) + 4S, per GPU) / average Jacobi launch "
                     "time: CUDA events the library records around the T back-to-back Jacobi launches of psn_smooth "
                     "(psn_ctx_set_smooth_events; iteration 1 also builds the smoothing cache, k_smooth_first), "
                     "recorded by each timed step's captured smoothing graph and averaged over the K timed steps "
                     "(K direct calls after the timed region with --no-graph), divided by T")
                    if t_v4 else
                    ("achieved = algorithmic bytes per launch / (smoothing half incl. the one-off cache prep) / T")}
    if dominant != sm_kern:
        roof["note"] += "; extraction dominated this config's step, see extract.frac"

    # per-pass roofline (SURVEY 8(d) per-kernel byte budgets, per GPU): counting reads the labels once,
    # the scan moves 24 B per voxel row, the emission writes the outputs (+ the face masks)
    nominal = 8000.0
    R = (N - 1) * (O - 1)
    out_bytes = 12 * P + 24 * Q + 4 * (P + 1) + 4 * S + P
    per_pass = {}
    for name, t_ms, byt, what in (
            ("k_count3", t_pass[0], V * b, "labels V*b (incl. the scan-header reset)"),
            ("k_scan", t_pass[1], 24 * R, "24 B per voxel row"),
            ("k_emit_band", t_pass[2], out_bytes, "outputs 12P + 24Q + 4(P+1) + 4S + P face masks")):
        gbs = byt / world / (t_ms * 1e-3) / 1e9 if t_ms > 0 else None
        per_pass[name] = {"ms": t_ms, "bytes": byt / world, "bytes_model": what, "gbs": gbs,
                          "frac": gbs / peak if gbs else None, "frac_nominal_8tbs": gbs / nominal if gbs else None}

    # ---------------------------------------------------------------- e2e through the public host-buffer API
    e2e = None
    if world == 1 and not args.no_e2e:
        host = torch.empty(labels.shape, dtype=labels.dtype, pin_memory=True)
        host.copy_(labels)
        sns = SurfaceNetsStream(psn, labels.shape, labels.dtype, sp, T, lam, d)
        for _ in range(sns.depth):                 # warm-up: sizes every slot
            sns.result(sns.submit(host))
        torch.cuda.synchronize()
        ke = max(1, args.e2e_steps)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sns.s_h2d)                       # before the first upload
        tickets = [sns.submit(host) for _ in range(ke)]
        sns.flush()                                # the last volume's compute (submit defers it by one)
        e1.record(sns.s_d2h)                       # after the last readback
        last = sns.result(tickets[-1])             # host outputs of the last volume are in host memory
        e1.synchronize()
        te = e0.elapsed_time(e1) / ke
        pts = last[0]
        state = {"h2d_bytes": sns.h2d_bytes, "d2h_bytes": sns.d2h_bytes}
        e2e = {"value": V / (te * 1e-3), "unit": "voxel/s", "h2d_bytes_per_step": int(state["h2d_bytes"]),
               "d2h_bytes_per_step": int(state["d2h_bytes"]), "ms_per_step": te, "steps": ke,
               "api": "paper_2401_14906_b200.psn.SurfaceNetsStream (per step: pinned host labels -> device, extract + "
                      "smooth, device -> pinned host points/quads/two-tuples; consecutive volumes overlap on "
                      "copy / compute / readback streams)",
               "timing": "CUDA events: first upload (copy stream) to last readback (readback stream), / steps"}
        del pts, last, sns
        del host, state

    # ---------------------------------------------------------------- CPU baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            n_layers = sample_layers(cfg, args.ref_voxels)
            lab_fn = lambda a, b_: labels[a:b_].cpu().numpy()   # noqa: E731
            tot, vox_tot, lab_host = 0.0, 0, None
            reps = 0
            while reps < 3 or (tot < args.cpu_seconds and reps < 64):   # ~10-30 s of CPU work
                dt, vox, (k0, k1), lab_host = oracle_sample(cfg, n_layers, labels_host=lab_host if lab_host is not None else lab_fn)
                tot += dt; vox_tot += vox; reps += 1
            cpu = {"value": vox_tot / tot, "unit": "voxel/s", "cores": 1, "kind": "oracle",
                   "sample": sample_text(cfg, k0, k1, vox, T, reps) + f"; {tot:.1f} s total",
                   "host": host_info()}
        except Exception as e:  # never fail the bench on the baseline leg
            cpu = {"value": None, "unit": "voxel/s", "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}

    if rank == 0:
        l2 = L2_BYTES
        line = {
            "metric": METRIC, "value": value, "unit": "voxel/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": {1: "u8", 2: "u16", 4: "u32"}[b] + "/f32", "data": "synthetic",
            "config": {"workload": WORKLOADS[cfg], "dims": [M, N, O], "label_bytes": b, "iterations": T,
                       "relaxation": lam, "constraint_voxels": d, "spacing": list(sp),
                       "parallelism": (f"z-slab x{world}" + {"points": " (layers cut to equal point counts)",
                                                             "c4": ", point-balanced smoothing re-partition (C4)",
                                                             "equal": " (equal layers)"}[args.partition]
                                       + (", halo: kernel peer pushes (NVLink, CUDA IPC)" if halo_peer
                                          else ", halo: NCCL point-to-point"))
                       if world > 1 else "single GPU",
                       "launch": "step replayed as 2 CUDA graphs (extraction, smoothing); per_pass from direct calls"
                       if graphs else "direct library calls",
                       "l2": ("inputs larger than L2 (%.2f GB labels, %.2f GB smoothing state)" % (V * b / 1e9, P * 28 / 1e9))
                       if V * b > l2 else "inputs fit in L2: L2 flushed (2x L2 written) before every timed step"},
            "counts": {"points": P, "quads": Q, "stencil": S},
            "extract": {"ms": t_ext, "voxels_per_s": ext_vps, "bytes_alg": b_ext, "gbs": ext_gbs, "frac": ext_gbs / world / peak,
                        "frac_nominal_8tbs": ext_gbs / world / nominal},
            "per_pass": per_pass,
            "smooth": {"ms": t_sm, "pt_iters_per_s": sm_ptit, "bytes_alg_per_iter": b_sm, "gbs": sm_gbs,
                       "frac": sm_gbs / world / peak, "frac_nominal_8tbs": sm_gbs / world / nominal},
            "roofline": roof,
            "gpu_launches": launches * K if world == 1 else None,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="psn", choices=["psn", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--partition", default="points", choices=["points", "c4", "equal"],
                    help="N > 1: 'points' = voxel-layer slabs cut to equal point counts (from the per-layer counts, "
                         "once) for extraction and smoothing; 'c4' = equal slabs + the per-step point-balanced "
                         "smoothing re-partition; 'equal' = equal slabs for both")
    ap.add_argument("--nccl-halo", action="store_true",
                    help="N > 1: smoothing halo exchange over NCCL point-to-point instead of the kernel's peer pushes")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-graph", action="store_true",
                    help="N = 1: call the library per step instead of replaying the step's CUDA graphs")
    ap.add_argument("--smooth-cache", action="store_true",
                    help="N = 1: the emission writes the packed smoothing cache next to the stencils and psn_smooth "
                         "skips k_smooth_prep8 (measured: c4 step -0.2 %%, extraction +3 %%; c5a step -1.6 %%)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="cpu_baseline: repeat the reference arm's sample window until this much CPU time")
    ap.add_argument("--ref-voxels", type=float, default=8e6,
                    help="oracle sample window per reference step (also the cpu_baseline window)")
    ap.add_argument("--check-launch", action="store_true",
                    help="bring up the N ranks (NCCL, or gloo without CUDA), check world == --gpus, print and exit")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N`: bring up N ranks through torchrun (one process per GPU)
        relaunch(args.gpus)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch N ranks for --gpus N")
        sys.exit(2)
    if args.check_launch:
        check_launch(rank, world, local_rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "reference":
            if rank == 0:
                run_reference(args, rank, world)
            return
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        try:
            run_psn(args, rank, world, local_rank)
        finally:
            dist.destroy_process_group()
        return
    if args.impl == "reference":
        run_reference(args, 0, 1)
    else:
        run_psn(args, 0, 1, 0)


def relaunch(n: int):
    """Re-exec this command under torch.distributed.run with n local ranks (127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    log("bench.py: launching", n, "ranks:", " ".join(cmd[1:]))
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def check_launch(rank, world, local_rank):
    """--check-launch: every rank joins the process group (NCCL on GPUs, gloo otherwise) and
    all-gathers its rank; rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist
    if world == 1:
        print(json.dumps({"n_gpus": 1, "ranks": [0], "backend": None}), flush=True)
        return
    use_nccl = torch.cuda.is_available() and torch.cuda.device_count() >= world
    if use_nccl:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dev = torch.device("cuda", local_rank)
    else:
        dist.init_process_group("gloo")
        dev = torch.device("cpu")
    try:
        t = torch.tensor([rank], dtype=torch.int64, device=dev)
        out = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        if rank == 0:
            print(json.dumps({"n_gpus": world, "ranks": [int(x.item()) for x in out],
                              "backend": "nccl" if use_nccl else "gloo"}), flush=True)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
