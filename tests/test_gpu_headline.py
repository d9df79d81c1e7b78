"""Parity at the benchmarked configuration (BASELINE config 3): 128^3, K=32,
Nt=10, the SURVEY §8(d) micro-benchmark recipe, run on the pad-100 engine the
bench times (``WShape<10,10>``).

The fixtures ``headline_128_{state,def}.npz`` come from the UNMODIFIED
reference (``tests/golden/make_golden.py --headline``, ~20 CPU-minutes per
objective) and hold, at full double precision: the energy, and for the
gradient, the GN HVP and the Newton HVP the Frobenius norm, Re<x, w>,
Re<x, r> against a seeded probe r, and 1000 seeded complex coefficients.

Tolerances: fp64 1e-10 relative (energy 1e-12); fp32 1e-4.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from golden_io import exists, headline_probe, load  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import blreg_oracle as O  # noqa: E402
import paper_1807_05117_b200 as B  # noqa: E402
from paper_1807_05117_b200 import spectral  # noqa: E402

_CACHE = {}


def _inputs():
    if "in" not in _CACHE:
        odom = O.Dom((128,) * 3, (32,) * 3, alpha=0.02, order=2)
        rng = np.random.default_rng(0)
        I0, I1 = O.band_image(odom, rng), O.band_image(odom, rng)
        v = O.smooth_vector_block(odom, rng, 0.5 / 128, decay=2.0)[None]
        w = O.smooth_vector_block(odom, rng, 0.5 / 128, decay=2.0)[None]
        _CACHE["in"] = (I0, I1, v, w)
    return _CACHE["in"]


def _check_vector(name, x, g, w, r, tol):
    x = x.detach().cpu().numpy().astype(np.complex128)
    idx = g["sample_idx"]
    ref_s = g[f"{name}_samples"]
    got_s = x.reshape(-1)[idx]
    assert np.linalg.norm(got_s - ref_s) <= tol * np.linalg.norm(ref_s), name
    ref_n = float(g[f"{name}_norm"])
    assert np.linalg.norm(x) == pytest.approx(ref_n, rel=tol), name
    # Re<x, w>, Re<x, r> (reference spectral.inner = Re vdot(b, a)); the
    # probe terms are bounded by |x - ref| |probe| (Cauchy-Schwarz)
    for key, probe in (("dot_w", w), ("dot_r", r)):
        got = float(np.real(np.vdot(probe, x)))
        assert abs(got - float(g[f"{name}_{key}"])) <= tol * ref_n * np.linalg.norm(probe), (name, key)


@pytest.mark.parametrize("dtype,tol,etol", [("float64", 1e-10, 1e-12), ("float32", 1e-4, 1e-5)])
@pytest.mark.parametrize("kind", ["def", "state"])
def test_headline_128(kind, dtype, tol, etol):
    name = f"headline_128_{kind}"
    if not exists(name):
        pytest.skip("fixture needs make_golden --headline")
    g = load(name)
    I0, I1, v, w = _inputs()
    dom = B.Domain((128,) * 3, (32,) * 3, alpha=0.02, order=2, dtype=dtype)
    assert dom.pad == (100, 100, 100)  # the engine instantiation the bench measures
    r, idx = headline_probe(v.shape)
    assert np.array_equal(idx, g["sample_idx"])
    cls = B.StateObjective if kind == "state" else B.DeformationObjective
    obj = cls(dom, I0, I1, B.ProblemConfig(sigma2=0.1, n_time_steps=10))
    vf = B.TimeFlow(dom, v, 10, True)
    wf = B.TimeFlow(dom, w, 10, True)
    assert obj.energy(vf) == pytest.approx(float(g["energy_direct"]), rel=etol)
    ev = obj.gradient(vf)
    assert ev.energy == pytest.approx(float(g["energy"]), rel=etol)
    assert ev.cache.substeps == int(g["substeps"])
    _check_vector("grad", ev.gradient.values, g, w, r, tol)
    _check_vector("hvp_gn", ev.hessian_vector(wf, gauss_newton=True).values, g, w, r, tol)
    _check_vector("hvp_newton", ev.hessian_vector(wf, gauss_newton=False).values, g, w, r, tol)
