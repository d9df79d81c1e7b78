"""Known-answer and property checks ported from the reference test-suite
(``pkg/tests/test_{spectral,transport,objectives,solver,gridops}.py``), run on
the sm_100a path.  Citations are to the reference test that each one ports.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import blreg_oracle as O  # noqa: E402
import paper_1807_05117_b200 as B  # noqa: E402
from paper_1807_05117_b200 import gridops, spectral, transport  # noqa: E402
from paper_1807_05117_b200.transport import TimeFlow  # noqa: E402


def np_(t):
    return t.detach().cpu().numpy()


def dc_flow(dom, c, n_steps=10):
    v = np.zeros((dom.ndim,) + dom.block_shape, complex)
    for ax, val in enumerate(c):
        v[(ax,) + (0,) * dom.ndim] = val
    return TimeFlow(dom, v[None], n_steps, True)


def test_symbol_value():  # test_spectral.py:179-185
    dom = B.Domain((64, 64), (16, 16), alpha=0.05, order=2)
    sym = spectral.metric_symbol(dom)
    f = dom.frequencies()
    expected = (1.0 + 0.05 * sum(2 * 64 * 64 * (1 - np.cos(2 * np.pi * k / 64)) for k in (f[0][3], f[1][-2]))) ** 2
    assert sym[3, -2] == pytest.approx(expected, rel=1e-14)
    c = np.zeros(dom.block_shape, complex)
    c[3, -2] = 1.0
    c[-3, 2] = 1.0
    out = np_(spectral.apply_helmholtz(dom, c))
    assert out[3, -2].real == pytest.approx(expected, rel=1e-13)


def test_include_project_roundtrip_3d():  # test_spectral.py:56-62
    dom = B.Domain((16, 12, 20), (4, 3, 5))
    rng = np.random.default_rng(0)
    c = O.random_vector_block(O.Dom(dom.shape, dom.bandwidth), rng)
    back = np_(spectral.project(dom, spectral.include(dom, c)))
    np.testing.assert_allclose(back, c, atol=1e-13)


def test_dc_translation_map():  # test_transport.py:88-98
    dom = B.Domain((32, 32), (8, 8))
    c = (0.03, -0.02)
    phi = np_(transport.integrate_forward_map(dc_flow(dom, c)))
    for ax in range(2):
        assert phi[-1][(ax, 0, 0)].real == pytest.approx(-c[ax], abs=1e-14)
        rest = phi[-1][ax].copy()
        rest[0, 0] = 0
        assert np.abs(rest).max() < 1e-14


def test_inverse_map_characteristics():  # test_transport.py:130-141
    dom = B.Domain((32, 32), (8, 8))
    c = (0.04, 0.01)
    psi, vol = transport.integrate_inverse_map_and_volume(dc_flow(dom, c))
    psi = np_(psi)
    t = np.arange(11) / 10
    for ax in range(2):
        np.testing.assert_allclose(psi[:, ax, 0, 0].real, (1 - t) * c[ax], atol=1e-14)
    assert np.abs(np_(vol)[:, 0, 0] - 1.0).max() < 1e-14


def test_divergence_free_preserves_volume():  # test_transport.py:120-128
    dom = B.Domain((32, 32), (8, 8))
    odom = O.Dom(dom.shape, dom.bandwidth)
    v = O.leray(odom, O.smooth_vector_block(odom, np.random.default_rng(3), 0.05))
    _, vol = transport.integrate_inverse_map_and_volume(TimeFlow(dom, v[None], 10, True))
    J = np_(spectral.include(dom, vol, check=False))
    assert np.abs(J - 1.0).max() < 1e-6


def test_cfl_formula_and_substeps():  # test_transport.py:58-79
    dom = B.Domain((64, 64), (16, 16))
    flow = dc_flow(dom, (1.0, 0.0))
    rep = transport.check_cfl(flow)
    assert rep.number == pytest.approx(6.4, rel=1e-12)
    assert rep.suggested_steps == 128
    assert transport.resolve_substeps(flow, 0.5, True) == 13
    with pytest.raises(transport.CFLViolation):
        transport.resolve_substeps(flow, 0.5, False)


def test_tangent_linearity():  # test_transport.py:187-195
    dom = B.Domain((24, 24), (6, 6))
    odom = O.Dom(dom.shape, dom.bandwidth)
    rng = np.random.default_rng(4)
    v = TimeFlow(dom, O.smooth_vector_block(odom, rng, 0.05)[None], 8, True)
    a = TimeFlow(dom, O.smooth_vector_block(odom, rng, 0.05)[None], 8, True)
    b = TimeFlow(dom, O.smooth_vector_block(odom, rng, 0.05)[None], 8, True)
    da = transport.integrate_state_tangents(v, a, with_inverse=False)[0]
    db = transport.integrate_state_tangents(v, b, with_inverse=False)[0]
    dab = transport.integrate_state_tangents(v, 2.0 * a - 3.0 * b, with_inverse=False)[0]
    np.testing.assert_allclose(np_(dab), np_(2 * da - 3 * db), atol=1e-13 * float(dab.abs().max()))


@pytest.fixture(scope="module")
def images():
    dom = B.Domain((32, 32), (8, 8), alpha=0.05)
    odom = O.Dom(dom.shape, dom.bandwidth, alpha=0.05)
    rng = np.random.default_rng(0)
    return dom, O.band_image(odom, rng), O.band_image(odom, rng)


@pytest.mark.parametrize("cls", [B.StateObjective, B.DeformationObjective])
def test_zero_velocity_gradient_is_endpoint_term(images, cls):  # test_objectives.py:73-82
    dom, I0, I1 = images
    cfg = B.ProblemConfig(sigma2=1.3, interp="fourier", image_grad="spectral", quadrature="simpson",
                          n_time_steps=32)
    ev = cls(dom, I0, I1, cfg).gradient(TimeFlow.zero(dom, 32))
    odom = O.Dom(dom.shape, dom.bandwidth, alpha=0.05)
    lam = -(2.0 / 1.3) * (I0 - I1)
    gI0 = O.include(odom, O.grad(odom, O.project(odom, I0)))
    expected = O.project(odom, lam[None] * gI0)
    np.testing.assert_allclose(np_(ev.gradient.values[0]), expected, rtol=0, atol=1e-10)


def test_formulations_agree_at_zero(images):  # test_objectives.py:221-230
    dom, I0, I1 = images
    a = B.StateObjective(dom, I0, I1, B.ProblemConfig()).gradient(TimeFlow.zero(dom)).gradient
    b = B.DeformationObjective(dom, I0, I1, B.ProblemConfig()).gradient(TimeFlow.zero(dom)).gradient
    scale = float(a.values.abs().max())
    assert float((a.values - b.values).abs().max()) <= 1e-10 * scale


@pytest.mark.parametrize("cls", [B.StateObjective, B.DeformationObjective])
def test_gn_curvature_bound(images, cls):  # test_objectives.py:169-181
    dom, I0, I1 = images
    odom = O.Dom(dom.shape, dom.bandwidth, alpha=0.05)
    rng = np.random.default_rng(17)
    obj = cls(dom, I0, I1, B.ProblemConfig(n_time_steps=10))
    ev = obj.gradient(TimeFlow(dom, O.smooth_vector_block(odom, rng, 0.05, 3.0)[None], 10, True))
    ws = [TimeFlow(dom, O.smooth_vector_block(odom, rng, 1.0, 1.0)[None], 10, True) for _ in range(3)]
    for w in ws:
        hw = ev.hessian_vector(w, gauss_newton=True)
        lw = w._like(spectral.apply_helmholtz(dom, w.values))
        assert transport.flow_inner(hw, w) >= (1.0 - 1e-8) * transport.flow_inner(lw, w)


@pytest.mark.parametrize("cls", [B.StateObjective, B.DeformationObjective])
def test_errors(images, cls):  # test_objectives.py:57-63, 194-201
    dom, I0, I1 = images
    with pytest.raises(ValueError):
        cls(dom, I0, I1, B.ProblemConfig(sigma2=1e-320)).gradient(TimeFlow.zero(dom))
    with pytest.raises(ValueError):
        cls(dom, I0[:-1], I1)
    bad = I0.copy()
    bad[0, 0] = np.nan
    with pytest.raises(ValueError):
        cls(dom, bad, I1)
    obj = cls(dom, I0, I1)
    odom = O.Dom(dom.shape, dom.bandwidth, alpha=0.05)
    v = TimeFlow(dom, O.smooth_vector_block(odom, np.random.default_rng(1), 0.03)[None], 10, True)
    ev = obj.gradient(v)
    ev.cache.velocity = 2.0 * v
    with pytest.raises(ValueError):
        ev.hessian_vector(v)


def test_pcg_known_answers():  # test_solver.py:23-72
    dom = B.Domain((16, 16), (4, 4), alpha=0.5, order=2)
    odom = O.Dom(dom.shape, dom.bandwidth, alpha=0.5)
    g = TimeFlow(dom, O.smooth_vector_block(odom, np.random.default_rng(0))[None], 10, True)

    def prec(f):
        return f._like(spectral.apply_inverse_helmholtz(dom, f.values))

    x, it, neg = B.pcg_solve(lambda f: f, TimeFlow.zero(dom), B.SolverConfig(), prec, "trapezoid")
    assert it == 0 and not neg
    x, it, neg = B.pcg_solve(lambda f: f._like(spectral.apply_helmholtz(dom, f.values)), g,
                             B.SolverConfig(), prec, "trapezoid")
    assert it == 1 and not neg
    np.testing.assert_allclose(np_(x.values[0]), np_(spectral.apply_inverse_helmholtz(dom, g.values[0])),
                               atol=1e-10)
    x, it, neg = B.pcg_solve(lambda f: -1.0 * f, g, B.SolverConfig(), prec, "trapezoid")
    assert neg and it == 0


def test_identical_images_converge_immediately():  # test_solver.py:97-105
    dom = B.Domain((32, 32), (8, 8))
    img = O.band_image(O.Dom(dom.shape, dom.bandwidth), np.random.default_rng(6))
    res = B.minimize(B.StateObjective(dom, img, img, B.ProblemConfig()), TimeFlow.zero(dom))
    assert res.status == "converged"
    assert res.records[0].energy == pytest.approx(0.0, abs=1e-14)


def test_jacobian_determinant_translation():  # test_gridops.py:156-161
    dom = B.Domain((32, 32), (8, 8))
    u = np.full((2, 32, 32), 0.1)
    assert np.abs(np_(gridops.jacobian_determinant(dom, u)) - 1.0).max() < 1e-14
