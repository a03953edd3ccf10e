"""Loader for the committed golden vectors (tests/golden/*.npz + golden_meta.json)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def meta():
    with open(os.path.join(GOLDEN, "golden_meta.json")) as fh:
        return json.load(fh)


def arrays(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))
