"""A/B builds of libpsn.so and interleaved per-pass timing (GPU box).

    python tools/ab.py build NAME [-DMACRO=VAL ...]      -> ab/libpsn_NAME.so
    python tools/ab.py run --libs base,new --configs c4,c3 --rounds 3
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(name, defines):
    from paper_2401_14906_b200 import build as b
    os.makedirs(os.path.join(ROOT, "ab"), exist_ok=True)
    out = os.path.join(ROOT, "ab", f"libpsn_{name}.so")
    cmd = ["nvcc", *b.NVCC_FLAGS, *defines, "-I", os.path.join(ROOT, "include"), "-I", os.path.join(b.HERE, "csrc"),
           "-o", out, b.SRC]
    subprocess.check_call(cmd)
    print(out)


def run(libs, configs, rounds, digest):
    res = {}
    for r in range(rounds):
        for cfg in configs:
            for lib in libs:
                env = dict(os.environ)
                env["PSN_LIB"] = os.path.join(ROOT, "ab", f"libpsn_{lib}.so") if lib != "default" else \
                    os.path.join(ROOT, "paper_2401_14906_b200", "libpsn.so")
                cmd = [sys.executable, os.path.join(ROOT, "tools", "pass_time.py"), "--config", cfg]
                if digest:
                    cmd.append("--digest")
                p = subprocess.run(cmd, capture_output=True, text=True, env=env)
                if p.returncode != 0:
                    print("FAIL", lib, cfg, p.stderr[-1500:], flush=True)
                    continue
                d = json.loads(p.stdout.strip().splitlines()[-1])
                res.setdefault((cfg, lib), []).append(d)
                print(json.dumps({"round": r, "lib": lib, **{k: v for k, v in d.items() if k != "lib"}}), flush=True)
    print("summary (median over rounds):")
    for (cfg, lib), ds in sorted(res.items()):
        f = lambda k: statistics.median(x[k] for x in ds)  # noqa: E731
        dig = {x.get("digest") for x in ds}
        print(f"{cfg:4s} {lib:12s} count {f('count_ms'):.4f} scan {f('scan_ms'):.4f} emit {f('emit_ms'):.4f} "
              f"total {f('total_ms'):.4f}  digest {dig if digest else ''}")


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3:])
    else:
        import argparse
        ap = argparse.ArgumentParser()
        ap.add_argument("cmd")
        ap.add_argument("--libs", default="default")
        ap.add_argument("--configs", default="c4")
        ap.add_argument("--rounds", type=int, default=3)
        ap.add_argument("--digest", action="store_true")
        a = ap.parse_args()
        run(a.libs.split(","), a.configs.split(","), a.rounds, a.digest)
