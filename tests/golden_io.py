"""Load the reference-generated golden vectors (tests/golden/make_golden.py)."""

import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load():
    arrays = np.load(os.path.join(HERE, "golden.npz"))
    with open(os.path.join(HERE, "golden.json")) as f:
        meta = json.load(f)
    return arrays, meta


def uniform(seed, n, d):
    """Same draw order as make_golden.uniform."""
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, (n, d)), rng.uniform(-1, 1, (n, d)), rng.uniform(-1, 1, (n, d)))
