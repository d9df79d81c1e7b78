"""Fused library entry points against their unfused compositions.

``blr_momentum_contract`` (backward momentum transport + summed node
contraction, used by the Gauss-Newton deformation HVP) must equal
``blr_momentum`` followed by ``blr_contract`` with weights, for both
contraction conventions, with and without the D(phi) node cache, in fp64 and
fp32.  The fused path never materializes the momentum node records and sums
the nodes in a different order, so agreement is to round-off.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1807_05117_b200 as B  # noqa: E402
from paper_1807_05117_b200 import _lib, transport  # noqa: E402
from paper_1807_05117_b200.spectral import ptr  # noqa: E402

import bench  # noqa: E402


def rel(a, b):
    a, b = a.detach().cpu().numpy(), b.detach().cpu().numpy()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-12), ("float32", 2e-5)])
@pytest.mark.parametrize("transposed", [0, 1])
@pytest.mark.parametrize("cached", [False, True])
@pytest.mark.parametrize("shape,K,nt", [((24, 24, 24), 6, 4), ((20, 16, 28), 5, 3)])
def test_momentum_contract_matches_composition(dtype, tol, transposed, cached, shape, K, nt):
    dom = B.Domain(shape, (K,) * 3, alpha=0.05, dtype=dtype)
    rng = np.random.default_rng(7)
    v = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.04, 2.0)[None], nt, True)
    rho_end = torch.as_tensor(bench.smooth_vector_block(dom, rng, 1.0, 1.5), device=dom.torch_device)
    rho_end = rho_end.to(dom.cdtype).contiguous()
    du_cache = torch.empty(transport.du_cache_shape(v, 1), dtype=dom.rdtype, device=dom.torch_device)
    phi = transport.integrate_forward_map(v, 1, du_cache)
    n = v.n_nodes
    weights = np.linspace(0.5, 1.5, n) / n
    w, keep = _lib.double_array(weights)
    h = dom.ctx().bind()
    cache = None
    if cached:  # fill the D(phi_i) cache through the unfused contraction (mode 1)
        cache = torch.empty((n, dom.ndim * dom.ndim) + dom.pad, dtype=dom.rdtype, device=dom.torch_device)
        scratch = torch.empty((dom.ndim,) + dom.block_shape, dtype=dom.cdtype, device=dom.torch_device)
        rho0 = transport.integrate_momentum(v, rho_end, 1)
        _lib.call("blr_contract", h, ptr(phi), ptr(rho0), n, w, transposed, ptr(cache), 1, ptr(scratch))
    mode = 2 if cached else 0
    rho = transport.integrate_momentum(v, rho_end, 1)
    ref = torch.empty((dom.ndim,) + dom.block_shape, dtype=dom.cdtype, device=dom.torch_device)
    _lib.call("blr_contract", h, ptr(phi), ptr(rho), n, w, transposed,
              ptr(cache) if cache is not None else None, mode, ptr(ref))
    out = torch.empty_like(ref)
    _lib.call("blr_momentum_contract", h, ptr(v.values), v.n_stored, v.n_steps, 1, ptr(rho_end), ptr(phi), w,
              transposed, ptr(cache) if cache is not None else None, mode, ptr(out))
    torch.cuda.synchronize()
    del keep
    assert rel(out, ref) < tol


def test_momentum_contract_rejects_missing_weights():
    dom = B.Domain((16, 16, 16), (4, 4, 4), alpha=0.05)
    v = B.TimeFlow.zero(dom)
    rho_end = torch.zeros((3,) + dom.block_shape, dtype=dom.cdtype, device=dom.torch_device)
    out = torch.empty_like(rho_end)
    with pytest.raises(ValueError, match="bad arguments"):
        _lib.call("blr_momentum_contract", dom.ctx().bind(), ptr(v.values), v.n_stored, v.n_steps, 1,
                  ptr(rho_end), None, None, 0, None, 0, ptr(out))


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("kind", ["def", "state"])
@pytest.mark.parametrize("N,K", [(128, 32), (64, 16), (40, 12)])
def test_fused_forward_projection_bit_identical(dtype, kind, N, K):
    """The fused y+x forward projection (blr_fwd2.cuh: one cluster per
    (output, kz) plane, DSMEM exchange, kz = 0 mirror symmetrization) performs
    the two-kernel path's arithmetic operation for operation: energy, gradient
    and GN / Newton HVPs must be bit-identical with it on and off."""
    dom = B.Domain((N,) * 3, (K,) * 3, alpha=0.02, order=2, dtype=dtype)
    rng = np.random.default_rng(11)
    I0, I1 = bench.band_image(dom, rng), bench.band_image(dom, rng)
    v = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / N, 2.0)[None], 4, True)
    w = B.TimeFlow(dom, bench.smooth_vector_block(dom, rng, 0.5 / N, 2.0)[None], 4, True)
    cls = B.DeformationObjective if kind == "def" else B.StateObjective
    out = {}
    try:
        for on in (0, 1):
            _lib.call("blr_set_fused_forward", on)
            obj = cls(dom, I0, I1, B.ProblemConfig(sigma2=0.1, n_time_steps=4))
            ev = obj.gradient(v)
            out[on] = (ev.energy, ev.gradient.values.clone(), ev.hessian_vector(w, True).values.clone(),
                       ev.hessian_vector(w, False).values.clone())
    finally:
        _lib.call("blr_set_fused_forward", 0)
    assert out[0][0] == out[1][0]
    for a, b in zip(out[0][1:], out[1][1:]):
        assert torch.equal(a, b)
