"""Loader for the committed golden fixtures (tests/golden/make_golden.py)."""
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def meta():
    with open(os.path.join(HERE, "golden.json")) as fh:
        return json.load(fh)


_arrays = None


def arrays():
    global _arrays
    if _arrays is None:
        _arrays = dict(np.load(os.path.join(HERE, "golden.npz")))
    return _arrays


def solve_case(name):
    for c in meta()["solves"]:
        if c["name"] == name:
            return c
    raise KeyError(name)
