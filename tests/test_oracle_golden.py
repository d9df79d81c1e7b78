"""Pin the CPU oracle against fixtures produced by the unmodified reference.

These run on the CPU (no GPU marker).  Tolerances: 1e-12 relative for
single spectral operations, 1e-11 for integrated trajectories and objective
outputs (rounding differences only: real-to-complex vs complex transforms).
"""

import numpy as np
import pytest

import blreg_oracle as O
from golden_io import dom_args, exists, load, rel

SPECTRAL = ["spectral_3d", "spectral_2d", "spectral_1d", "spectral_nyq"]


def mkdom(g, pad=None):
    return O.Dom(**dom_args(g), pad=pad)


@pytest.mark.parametrize("name", SPECTRAL)
@pytest.mark.parametrize("pad_mode", ["ref", "min"])
def test_spectral(name, pad_mode):
    g = load(name)
    base = mkdom(g)
    pad = None if pad_mode == "ref" else tuple(3 * k + 1 for k in base.bandwidth)
    dom = mkdom(g, pad)
    assert rel(O.include(dom, g["a"]), g["include_a"]) < 1e-13
    assert rel(O.project(dom, g["f"]), g["project_f"]) < 1e-13
    assert rel(O.conv_matvec(dom, g["M"], g["a"]), g["matvec"]) < 1e-12
    assert rel(O.conv_matvec(dom, g["M"], g["a"], transpose=True), g["matvec_t"]) < 1e-12
    assert rel(O.conv_scalar(dom, g["s"], g["s"]), g["conv_s"]) < 1e-12
    assert rel(O.helmholtz(dom, g["a"]), g["helm"]) < 1e-15
    assert rel(O.inv_helmholtz(dom, g["a"]), g["ihelm"]) < 1e-15
    assert rel(O.leray(dom, g["a"]), g["leray"]) < 1e-15
    assert O.max_abs(dom, g["a"][0]) == pytest.approx(float(g["max_abs"]), rel=1e-14)
    assert O.inner(g["a"], 1.5 * g["a"] + 0.25 * g["M"][0]) == pytest.approx(
        float(g["inner_as"]), rel=1e-14)


@pytest.mark.parametrize("name", ["rhs_3d", "rhs_2d"])
def test_rhs(name):
    g = load(name)
    dom = mkdom(g)
    assert rel(O.rhs_map(dom, g["u"], g["v"]), g["map"]) < 1e-12
    assert rel(O.rhs_map_tangent(dom, g["u"], g["du"], g["v"], g["dv"]), g["map_t"]) < 1e-12
    assert rel(O.rhs_volume(dom, g["J"], g["v"]), g["vol"]) < 1e-12
    assert rel(O.rhs_volume_tangent(dom, g["J"], g["dJ"], g["v"], g["dv"]), g["vol_t"]) < 1e-12
    assert rel(O.rhs_momentum(dom, g["rho"], g["v"]), g["mom"]) < 1e-12
    b, t = O.rhs_momentum_pair(dom, g["rho"], g["drho"], g["v"], g["dv"])
    assert rel(b, g["pair_base"]) < 1e-12 and rel(t, g["pair_tan"]) < 1e-12
    _, t = O.rhs_momentum_pair(dom, g["rho"], g["drho"], g["v"], None)
    assert rel(t, g["pair_gn_tan"]) < 1e-12


@pytest.mark.parametrize("name", ["transport_3d", "transport_3d_sub", "transport_2d_ns"])
def test_transport(name):
    g = load(name)
    dom = mkdom(g)
    ns, sub, st = int(g["n_steps"]), int(g["substeps"]), bool(g["stationary"])
    v = O.Flow(dom, g["v"], ns, st)
    dv = O.Flow(dom, g["dv"], ns, st)
    assert O.cfl(v)[0] == pytest.approx(float(g["cfl_number"]), rel=1e-13)
    assert rel(O.forward_map(v, sub), g["phi"]) < 1e-11
    psi, vol = O.inverse_map_and_volume(v, sub)
    assert rel(psi, g["psi"]) < 1e-11 and rel(vol, g["vol"]) < 1e-11
    dphi, dpsi, dvol = O.state_tangents(v, dv, sub)
    assert rel(dphi, g["dphi"]) < 1e-11
    assert rel(dpsi, g["dpsi"]) < 1e-11 and rel(dvol, g["dvol"]) < 1e-11
    assert rel(O.momentum(v, g["rho1"], sub), g["rho"]) < 1e-11
    r, dr = O.momentum_tangent(v, dv, g["rho1"], g["drho1"], sub, False)
    assert rel(r, g["pair_rho"]) < 1e-11 and rel(dr, g["pair_drho"]) < 1e-11
    _, dr = O.momentum_tangent(v, dv, g["rho1"], g["drho1"], sub, True)
    assert rel(dr, g["pair_drho_gn"]) < 1e-11


@pytest.mark.parametrize("name", ["grid_3d", "grid_2d"])
def test_gridops(name):
    g = load(name)
    dom = mkdom(g)
    for interp in ("linear", "cubic", "nearest"):
        assert rel(O.warp(dom, g["img"], g["disp"], interp), g[f"warp_{interp}"]) < 1e-14
    assert rel(O.grid_grad(dom, g["img"], "central"), g["grad_central"]) < 1e-14
    assert rel(O.grid_grad(dom, g["img"], "spectral"), g["grad_spectral"]) < 1e-13
    assert rel(O.jacobian_det(dom, g["disp"]), g["jdet"]) < 1e-14


OBJ = ["obj_3d", "obj_3d_cubic_gamma", "obj_3d_direct_spec", "obj_2d", "obj_2d_ns",
       "obj_2d_refine"]


def problem_of(g):
    return O.Problem(sigma2=float(g["sigma2"]), gamma=int(g["gamma"]),
                     n_time_steps=int(g["n_steps"]), interp=str(g["interp"]),
                     image_grad=str(g["image_grad"]), quadrature=str(g["quadrature"]),
                     contraction=str(g["contraction"]))


@pytest.mark.parametrize("name", OBJ)
@pytest.mark.parametrize("kind", ["state", "def"])
def test_objective(name, kind):
    g = load(name)
    dom = mkdom(g)
    cfg = problem_of(g)
    st = bool(g["stationary"])
    v = O.Flow(dom, g["v"], cfg.n_time_steps, st)
    w = O.Flow(dom, g["w"], cfg.n_time_steps, st)
    obj = O.OracleObjective(dom, g["I0"], g["I1"], cfg, kind="state" if kind == "state" else "deformation")
    assert obj.energy(v) == pytest.approx(float(g[f"{kind}_energy"]), rel=1e-12)
    ev = obj.gradient(v)
    assert ev.substeps == int(g[f"{kind}_substeps"])
    assert ev.energy == pytest.approx(float(g[f"{kind}_grad_energy"]), rel=1e-12)
    assert ev.reg_energy == pytest.approx(float(g[f"{kind}_reg_energy"]), rel=1e-12)
    assert rel(ev.gradient.values, g[f"{kind}_grad"]) < 1e-10
    assert rel(ev.forward[-1], g[f"{kind}_forward_end"]) < 1e-11
    assert rel(obj.hessian_vector(ev, w, True).values, g[f"{kind}_hvp_gn"]) < 1e-10
    assert rel(obj.hessian_vector(ev, w, False).values, g[f"{kind}_hvp_newton"]) < 1e-10


@pytest.mark.slow
@pytest.mark.skipif(not exists("checksum_64"), reason="fixture needs make_golden --slow")
@pytest.mark.parametrize("kind", ["state", "def"])
def test_checksum_64(kind):
    g = load("checksum_64")
    dom = O.Dom((64,) * 3, (16,) * 3, alpha=0.02, order=2)
    rng = np.random.default_rng(0)
    I0, I1 = O.band_image(dom, rng), O.band_image(dom, rng)
    v = O.Flow(dom, O.smooth_vector_block(dom, rng, 0.5 / 64, decay=2.0)[None], 10, True)
    w = O.Flow(dom, O.smooth_vector_block(dom, rng, 0.5 / 64, decay=2.0)[None], 10, True)
    obj = O.OracleObjective(dom, I0, I1, O.Problem(sigma2=0.1), "state" if kind == "state" else "deformation")
    ev = obj.gradient(v)
    assert ev.energy == pytest.approx(float(g[f"{kind}_energy"]), rel=1e-12)
    hw = obj.hessian_vector(ev, w, True).values
    assert np.linalg.norm(hw) == pytest.approx(float(g[f"{kind}_hvp_norm"]), rel=1e-10)


@pytest.mark.parametrize("name", ["headline_128_state", "headline_128_def", "config2_64_state",
                                  "config2_64_def"])
def test_headline_probe_matches_fixture(name):
    """The GPU tests regenerate the seeded probe / sample indices; they must be
    the ones the reference-side generator used."""
    if not exists(name):
        pytest.skip("fixture needs make_golden --headline / --config2")
    from golden_io import headline_probe

    g = load(name)
    shape = (1, 3, 65, 65, 65) if name.startswith("headline") else (1, 3, 33, 33, 33)
    _, idx = headline_probe(shape)
    assert np.array_equal(idx, g["sample_idx"])
