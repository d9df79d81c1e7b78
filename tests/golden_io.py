"""Loading helpers for the reference-generated fixtures in ``tests/golden``."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def exists(name):
    return os.path.exists(os.path.join(GOLDEN, f"{name}.npz"))


def dom_args(g):
    return dict(shape=tuple(int(x) for x in g["shape"]),
                bandwidth=tuple(int(x) for x in g["bandwidth"]),
                alpha=float(g["alpha"]), order=int(g["order"]), symbol=str(g["symbol"]))


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.linalg.norm(b.ravel())
    num = np.linalg.norm((a - b).ravel())
    return num / den if den > 0 else num
