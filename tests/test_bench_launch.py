"""bench.py's launcher (CPU, gloo): `python bench.py --gpus N` alone brings up N ranks through
torch.distributed.run (127.0.0.1 rendezvous), and a launch whose world size differs from --gpus
is refused instead of silently measuring another N."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None); e.pop("RANK", None); e.pop("LOCAL_RANK", None)
    e["CUDA_VISIBLE_DEVICES"] = ""       # the CPU path (gloo) even on a GPU box
    if env:
        e.update(env)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=240, env=e, cwd=ROOT)


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_flag_launches_n_ranks(n):
    r = _run(["--gpus", str(n), "--check-launch"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line == {"n_gpus": n, "ranks": list(range(n)), "backend": "gloo"}


def test_world_size_mismatch_is_refused():
    r = _run(["--gpus", "2", "--check-launch"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=1" in r.stderr
