"""bench.py's JSON line carries every key of the measurement contract (c1, a few steps): the metric /
unit of BASELINE.json, the timing fields, roofline, per_pass, cpu_baseline (oracle, host info), e2e
(host buffers, bytes per step), gpu_launches and clocks -- and the reference arm prints its line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_bench_line_keys():
    d = _line(["--config", "c1", "--steps", "3", "--warmup", "3", "--e2e-steps", "2", "--cpu-seconds", "0.5"])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["metric"] == base["metric"] and d["unit"] == "voxel/s" and d["higher_is_better"] is True
    for k in ("value", "n_gpus", "steps", "warmup", "ms_per_step", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "per_pass", "cpu_baseline", "e2e", "gpu_launches", "clocks", "extract", "smooth"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"].startswith("c1")
    ro = d["roofline"]
    assert ro["bound"] == "hbm" and ro["unit"] == "GB/s" and ro["peak"] > 0 and abs(ro["frac"] - ro["achieved"] / ro["peak"]) < 1e-9
    assert set(d["per_pass"]) == {"k_count3", "k_scan", "k_emit_band"}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] > 0 and cb["host"]["nproc"] >= 1
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 32 ** 3 * 2 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "3"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
