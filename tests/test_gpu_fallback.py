"""The cuFFT (v1) path: pad lengths the fused pad engine does not support.

The pad engine covers the 7-smooth lengths in ``blr_fft.cuh``; any other pad
(here the reference's own ``next_fast_len(4K+1)`` choices such as 18 or 36)
falls back to cuFFT 3-D transforms with scatter / gather kernels.  The
fallback must give the same objective values as the reference fixtures, and
it must honour the engine-only shortcuts: the final-node-only forward
tangent (``blr_state_tangents`` bit 3) and ``blr_momentum_contract``.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from golden_io import dom_args, load, rel  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1807_05117_b200 as B  # noqa: E402
from paper_1807_05117_b200.domain import ENGINE_PADS  # noqa: E402
from paper_1807_05117_b200.objectives import (DeformationObjective, ProblemConfig,  # noqa: E402
                                              StateObjective)


def np_(t):
    return t.detach().cpu().numpy()


def reference_pad(K):
    """next_fast_len(4K+1) as the reference picks it (spectral.py:142-145): the
    smallest 2,3,5,7,11-smooth length, here never an engine length."""
    p = 4 * K + 1
    while True:
        r = p
        for f in (2, 3, 5, 7, 11):
            while r % f == 0:
                r //= f
        if r == 1 and p not in ENGINE_PADS:
            return p
        p += 1


def odd_pad(K):
    """Smallest odd length >= 3K+1 that is not an engine length: odd real sizes
    put cache slices at 8-byte offsets (cuFFT needs 16-byte aligned reals)."""
    p = 3 * K + 1
    while p % 2 == 0 or p in ENGINE_PADS:
        p += 1
    return p


@pytest.mark.parametrize("name", ["obj_3d", "obj_2d"])
@pytest.mark.parametrize("kind", ["state", "def"])
@pytest.mark.parametrize("padf", [reference_pad, odd_pad])
def test_objective_on_cufft_path(name, kind, padf):
    g = load(name)
    args = dom_args(g)
    pad = tuple(padf(k) for k in args["bandwidth"])
    dom = B.Domain(**args, pad=pad)
    assert not any(p in ENGINE_PADS for p in pad if p > 1)
    cfg = ProblemConfig(sigma2=float(g["sigma2"]), gamma=int(g["gamma"]), n_time_steps=int(g["n_steps"]),
                        interp=str(g["interp"]), image_grad=str(g["image_grad"]),
                        quadrature=str(g["quadrature"]), contraction=str(g["contraction"]))
    st = bool(g["stationary"])
    cls = StateObjective if kind == "state" else DeformationObjective
    obj = cls(dom, g["I0"], g["I1"], cfg)
    v = B.TimeFlow(dom, g["v"], cfg.n_time_steps, st)
    w = B.TimeFlow(dom, g["w"], cfg.n_time_steps, st)
    ev = obj.gradient(v)
    assert rel(np_(ev.gradient.values), g[f"{kind}_grad"]) < 1e-10
    assert rel(np_(ev.hessian_vector(w, gauss_newton=True).values), g[f"{kind}_hvp_gn"]) < 1e-10
    assert rel(np_(ev.hessian_vector(w, gauss_newton=False).values), g[f"{kind}_hvp_newton"]) < 1e-10


@pytest.mark.parametrize("N,K,alt", [(136, 64, 198), (128, 32, 98), (48, 20, 66), (40, 16, 54)])
def test_engine_lengths_match_cufft(N, K, alt):
    """The largest engine lengths (196 = 14x14, 100 = the benchmarked
    128^3/K=32 instantiation, 64, 50) against the cuFFT path
    at another exact pad: both are the exact truncated convolution, so energy,
    gradient and GN / Newton HVPs agree to round-off (3-D, deformation)."""
    import bench

    res = {}
    for pad in ("engine", alt):
        dom = B.Domain((N,) * 3, (K,) * 3, alpha=0.02, **({} if pad == "engine" else {"pad": (alt,) * 3}))
        if pad == "engine":
            assert dom.pad[0] in ENGINE_PADS
        r = np.random.default_rng(3)
        I0, I1 = bench.band_image(dom, r), bench.band_image(dom, r)
        v = B.TimeFlow(dom, bench.smooth_vector_block(dom, r, 0.5 / N, 2.0)[None], 4, True)
        w = B.TimeFlow(dom, bench.smooth_vector_block(dom, r, 0.5 / N, 2.0)[None], 4, True)
        obj = DeformationObjective(dom, I0, I1, ProblemConfig(sigma2=0.1, n_time_steps=4))
        ev = obj.gradient(v)
        res[pad] = (ev.energy, np_(ev.gradient.values), np_(ev.hessian_vector(w, True).values),
                    np_(ev.hessian_vector(w, False).values))
    a, b = res["engine"], res[alt]
    assert a[0] == pytest.approx(b[0], rel=1e-12)
    for x, y in zip(a[1:], b[1:]):
        assert rel(x, y) < 1e-10
