"""Load the reference-generated golden fixtures (tests/golden/golden.npz)."""
import os

import numpy as np

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")
_CACHE = {}


def golden():
    if "g" not in _CACHE:
        _CACHE["g"] = dict(np.load(_PATH))
    return _CACHE["g"]


def tt(key):
    g = golden()
    n = int(g[f"{key}/n"])
    return [np.asfortranarray(g[f"{key}/{k}"]) for k in range(n)]
