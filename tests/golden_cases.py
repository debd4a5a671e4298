"""Parser for tests/golden/worked_cases.txt (cited worked cases)."""
import os

import numpy as np

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "worked_cases.txt")


def load():
    cases, cur = {}, None
    with open(_PATH) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, _, rest = line.partition(" ")
            if key == "case":
                cur = {"name": rest, "sets": [], "rows": [], "mquads": []}
            elif key == "end":
                cases[cur["name"]] = cur
                cur = None
            elif key == "set":
                cur["sets"].append([int(x) for x in rest.split()])
            elif key == "row":
                cur["rows"].append(rest)
            elif key == "mquad":
                cur["mquads"].append(rest)
            else:
                cur[key] = rest
    return cases


def volume(case, dtype=np.uint16):
    M, N, O = (int(x) for x in case["dims"].split())
    fill = int(case.get("fill", "0"))
    a = np.full((O, N, M), fill, dtype)
    for i, j, k, v in case["sets"]:
        a[k, j, i] = v
    return a
