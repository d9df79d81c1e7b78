"""GPU parity: the sm_100a path against fixtures produced by the unmodified
reference (``tests/golden``) and against the CPU oracle.

Tolerances: spectral ops 1e-12 relative; trajectories
1e-11; gradient and Hessian-vector products 1e-10 relative (Frobenius) in
fp64 and 1e-4 in fp32; energies 1e-12 (fp64).  The pad grid is the smallest
7-smooth size >= 3K+1 (the reference uses next_fast_len(4K+1)); agreement at
these tolerances is the evidence that the smaller pad is exact.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from golden_io import dom_args, load, rel  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1807_05117_b200 as B  # noqa: E402
from paper_1807_05117_b200 import gridops, spectral, transport  # noqa: E402
from paper_1807_05117_b200.objectives import (DeformationObjective, ProblemConfig,  # noqa: E402
                                              StateObjective)


def np_(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def gdom(g, **kw):
    return B.Domain(**dom_args(g), **kw)


@pytest.mark.parametrize("name", ["spectral_3d", "spectral_2d", "spectral_1d", "spectral_nyq"])
def test_spectral(name):
    g = load(name)
    dom = gdom(g)
    assert rel(np_(spectral.include(dom, g["a"])), g["include_a"]) < 1e-13
    assert rel(np_(spectral.project(dom, g["f"])), g["project_f"]) < 1e-13
    assert rel(np_(spectral.conv_matvec(dom, g["M"], g["a"])), g["matvec"]) < 1e-12
    assert rel(np_(spectral.conv_matvec(dom, g["M"], g["a"], transpose=True)), g["matvec_t"]) < 1e-12
    assert rel(np_(spectral.conv_scalar(dom, g["s"], g["s"])), g["conv_s"]) < 1e-12
    assert rel(np_(spectral.apply_helmholtz(dom, g["a"])), g["helm"]) < 1e-14
    assert rel(np_(spectral.apply_inverse_helmholtz(dom, g["a"])), g["ihelm"]) < 1e-14
    assert rel(np_(spectral.make_divergence_free(dom, g["a"])), g["leray"]) < 1e-14
    assert spectral.max_abs(dom, g["a"][0]) == pytest.approx(float(g["max_abs"]), rel=1e-13)
    assert spectral.inner(spectral.as_band(dom, g["a"]),
                          spectral.as_band(dom, 1.5 * g["a"] + 0.25 * g["M"][0]), dom) == \
        pytest.approx(float(g["inner_as"]), rel=1e-13)


def test_include_rejects_broken_symmetry():
    dom = B.Domain((16, 16), (4, 4))
    c = np.zeros(dom.block_shape, complex)
    c[1, 0] = 1.0  # no conjugate partner
    with pytest.raises(ValueError):
        spectral.include(dom, c)


@pytest.mark.parametrize("name", ["transport_3d", "transport_3d_sub", "transport_2d_ns"])
def test_transport(name):
    g = load(name)
    dom = gdom(g)
    ns, sub, st = int(g["n_steps"]), int(g["substeps"]), bool(g["stationary"])
    v = B.TimeFlow(dom, g["v"], ns, st)
    dv = B.TimeFlow(dom, g["dv"], ns, st)
    assert transport.check_cfl(v).number == pytest.approx(float(g["cfl_number"]), rel=1e-12)
    cache = torch.empty(transport.du_cache_shape(v, sub), dtype=dom.rdtype, device="cuda")
    phi = transport.integrate_forward_map(v, sub, cache)
    assert rel(np_(phi), g["phi"]) < 1e-11
    psi, vol = transport.integrate_inverse_map_and_volume(v, sub)
    assert rel(np_(psi), g["psi"]) < 1e-11 and rel(np_(vol), g["vol"]) < 1e-11
    dphi, dpsi, dvol = transport.integrate_state_tangents(v, dv, sub)
    assert rel(np_(dphi), g["dphi"]) < 1e-11
    assert rel(np_(dpsi), g["dpsi"]) < 1e-11 and rel(np_(dvol), g["dvol"]) < 1e-11
    dphi_c, _, _ = transport.integrate_state_tangents(v, dv, sub, with_inverse=False, du_cache=cache)
    assert rel(np_(dphi_c), g["dphi"]) < 1e-11
    assert rel(np_(transport.integrate_momentum(v, g["rho1"], sub)), g["rho"]) < 1e-11
    r, dr = transport.integrate_momentum_tangent(v, dv, g["rho1"], g["drho1"], sub, False)
    assert rel(np_(r), g["pair_rho"]) < 1e-11 and rel(np_(dr), g["pair_drho"]) < 1e-11
    _, dr = transport.integrate_momentum_tangent(v, dv, g["rho1"], g["drho1"], sub, True)
    assert rel(np_(dr), g["pair_drho_gn"]) < 1e-11


@pytest.mark.parametrize("name", ["grid_3d", "grid_2d"])
def test_gridops(name):
    g = load(name)
    dom = gdom(g)
    for interp in ("linear", "cubic", "nearest"):
        out = np_(gridops.warp(dom, g["img"], g["disp"], interp))
        assert rel(out, g[f"warp_{interp}"]) < (1e-12 if interp == "cubic" else 1e-14), interp
    assert rel(np_(gridops.spatial_gradient(dom, g["img"], "central")), g["grad_central"]) < 1e-14
    assert rel(np_(gridops.spatial_gradient(dom, g["img"], "spectral")), g["grad_spectral"]) < 1e-12
    assert rel(np_(gridops.jacobian_determinant(dom, g["disp"])), g["jdet"]) < 1e-14


OBJ = ["obj_3d", "obj_3d_cubic_gamma", "obj_3d_direct_spec", "obj_2d", "obj_2d_ns", "obj_2d_refine"]


def problem_of(g):
    return ProblemConfig(sigma2=float(g["sigma2"]), gamma=int(g["gamma"]),
                         n_time_steps=int(g["n_steps"]), interp=str(g["interp"]),
                         image_grad=str(g["image_grad"]), quadrature=str(g["quadrature"]),
                         contraction=str(g["contraction"]))


@pytest.mark.parametrize("name", OBJ)
@pytest.mark.parametrize("kind", ["state", "def"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_objective(name, kind, dtype):
    g = load(name)
    dom = gdom(g, dtype=dtype)
    cfg = problem_of(g)
    st = bool(g["stationary"])
    cls = StateObjective if kind == "state" else DeformationObjective
    obj = cls(dom, g["I0"], g["I1"], cfg)
    v = B.TimeFlow(dom, g["v"], cfg.n_time_steps, st)
    w = B.TimeFlow(dom, g["w"], cfg.n_time_steps, st)
    tol_e, tol_g = (1e-12, 1e-10) if dtype == "float64" else (1e-5, 1e-4)
    assert obj.energy(v) == pytest.approx(float(g[f"{kind}_energy"]), rel=tol_e)
    ev = obj.gradient(v)
    assert ev.cache.substeps == int(g[f"{kind}_substeps"])
    assert ev.energy == pytest.approx(float(g[f"{kind}_grad_energy"]), rel=tol_e)
    assert ev.reg_energy == pytest.approx(float(g[f"{kind}_reg_energy"]), rel=tol_e)
    assert rel(np_(ev.gradient.values), g[f"{kind}_grad"]) < tol_g
    assert rel(np_(ev.cache.forward[-1]), g[f"{kind}_forward_end"]) < tol_g
    hgn = ev.hessian_vector(w, gauss_newton=True)
    assert rel(np_(hgn.values), g[f"{kind}_hvp_gn"]) < tol_g
    hn = ev.hessian_vector(w, gauss_newton=False)
    assert rel(np_(hn.values), g[f"{kind}_hvp_newton"]) < tol_g
    # repeated products on one evaluation are deterministic
    assert torch.equal(ev.hessian_vector(w, gauss_newton=True).values, hgn.values)
