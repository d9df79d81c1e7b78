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


N_SAMPLES = 1000


def headline_probe(shape):
    """Seeded probe vector and coefficient-sample indices of the full-precision
    fixtures (must match ``make_golden.headline_probe``; checked on the CPU by
    ``test_oracle_golden.test_headline_probe_matches_fixture``)."""
    rng = np.random.default_rng(20260)
    r = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    idx = np.sort(rng.choice(int(np.prod(shape)), N_SAMPLES, replace=False))
    return r, idx
