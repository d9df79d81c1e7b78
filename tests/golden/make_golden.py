"""Generate golden fixtures by running the UNMODIFIED reference ``blreg``.

Run in the build container (where ``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--slow]

Every fixture stores the reference's inputs and outputs for one hot-path
operation family as an ``.npz`` next to this script.  The fixtures travel to
the GPU box; ``/root/reference`` does not.  ``--slow`` additionally records
the config-1 registration traces (2-D 64², K=16; ~3 CPU minutes) and the 3-D
64³/K=16 per-op checksums (~2 CPU minutes).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, f"{REF}/src")
sys.path.insert(0, f"{REF}/tests")
sys.dont_write_bytecode = True

from blreg import gridops, spectral, transport  # noqa: E402
from blreg.domain import Domain  # noqa: E402
from blreg.objectives import DeformationObjective, ProblemConfig, StateObjective  # noqa: E402
from blreg.solver import SolverConfig, minimize  # noqa: E402
from blreg.synthesis import synthesize_pair  # noqa: E402
from blreg.transport import TimeFlow  # noqa: E402
from helpers import (band_image, random_scalar_block, random_vector_block,  # noqa: E402
                     smooth_flow, smooth_vector_block)

OUT = os.path.dirname(os.path.abspath(__file__))


def dom_meta(dom: Domain) -> dict:
    return dict(shape=np.array(dom.shape), bandwidth=np.array(dom.bandwidth),
                alpha=dom.alpha, order=dom.order, symbol=dom.symbol)


def save(name, **arrays):
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def spectral_case(name, dom, seed):
    rng = np.random.default_rng(seed)
    d = dom.ndim
    a = random_vector_block(dom, rng)
    s = random_scalar_block(dom, rng)
    M = np.stack([random_vector_block(dom, rng) for _ in range(d)])
    f = rng.standard_normal((2,) + dom.shape)
    save(name, **dom_meta(dom), a=a, s=s, M=M, f=f,
         include_a=spectral.include(dom, a),
         project_f=spectral.project(dom, f),
         matvec=spectral.conv_matvec(dom, M, a),
         matvec_t=spectral.conv_matvec(dom, M, a, transpose=True),
         conv_s=spectral.conv_scalar(dom, s, s),
         helm=spectral.apply_helmholtz(dom, a),
         ihelm=spectral.apply_inverse_helmholtz(dom, a),
         leray=spectral.make_divergence_free(dom, a),
         max_abs=spectral.max_abs(dom, a[0]),
         inner_as=spectral.inner(a, 1.5 * a + 0.25 * M[0]))


def rhs_case(name, dom, seed):
    rng = np.random.default_rng(seed)
    u = smooth_vector_block(dom, rng, 0.05)
    du = smooth_vector_block(dom, rng, 0.05)
    v = smooth_vector_block(dom, rng, 0.05)
    dv = smooth_vector_block(dom, rng, 0.05)
    J = random_scalar_block(dom, rng, 0.01)
    J[(0,) * dom.ndim] = 1.0
    dJ = random_scalar_block(dom, rng, 0.01)
    rho = smooth_vector_block(dom, rng, 1.0)
    drho = smooth_vector_block(dom, rng, 1.0)
    mp = transport._momentum_pair_rhs(dom, rho, drho, v, dv)
    mpg = transport._momentum_pair_rhs(dom, rho, drho, v, None)
    save(name, **dom_meta(dom), u=u, du=du, v=v, dv=dv, J=J, dJ=dJ, rho=rho, drho=drho,
         map=transport._map_rhs(dom, u, v),
         map_t=transport._map_tangent_rhs(dom, u, du, v, dv),
         vol=transport._volume_rhs(dom, J, v),
         vol_t=transport._volume_tangent_rhs(dom, J, dJ, v, dv),
         mom=transport._momentum_rhs(dom, rho, v),
         pair_base=mp[0], pair_tan=mp[1], pair_gn_tan=mpg[1])


def transport_case(name, dom, seed, n_steps, substeps, stationary):
    rng = np.random.default_rng(seed)
    v = smooth_flow(dom, rng, amp=0.08, n_steps=n_steps, stationary=stationary)
    dv = smooth_flow(dom, rng, amp=0.08, n_steps=n_steps, stationary=stationary)
    rho1 = smooth_vector_block(dom, rng, 1.0)
    drho1 = smooth_vector_block(dom, rng, 1.0)
    phi = transport.integrate_forward_map(v, substeps)
    psi, vol = transport.integrate_inverse_map_and_volume(v, substeps)
    dphi, dpsi, dvol = transport.integrate_state_tangents(v, dv, substeps)
    rho = transport.integrate_momentum(v, rho1, substeps)
    r_n, dr_n = transport.integrate_momentum_tangent(v, dv, rho1, drho1, substeps, False)
    _, dr_gn = transport.integrate_momentum_tangent(v, dv, rho1, drho1, substeps, True)
    save(name, **dom_meta(dom), n_steps=n_steps, substeps=substeps, stationary=stationary,
         v=v.values, dv=dv.values, rho1=rho1, drho1=drho1,
         phi=phi, psi=psi, vol=vol, dphi=dphi, dpsi=dpsi, dvol=dvol, rho=rho,
         pair_rho=r_n, pair_drho=dr_n, pair_drho_gn=dr_gn,
         cfl_number=transport.check_cfl(v).number)


def grid_case(name, dom, seed):
    rng = np.random.default_rng(seed)
    img = band_image(dom, rng)
    disp = spectral.include(dom, smooth_vector_block(dom, rng, 3.0 / min(dom.shape)))
    out = dict(img=img, disp=disp)
    for interp in ("linear", "cubic", "nearest"):
        out[f"warp_{interp}"] = gridops.warp(dom, img, disp, interp=interp)
    out["grad_central"] = gridops.spatial_gradient(dom, img, "central")
    out["grad_spectral"] = gridops.spatial_gradient(dom, img, "spectral")
    out["jdet"] = gridops.jacobian_determinant(dom, disp)
    save(name, **dom_meta(dom), **out)


def objective_case(name, dom, seed, cfg: ProblemConfig, stationary=True, amp=0.05):
    rng = np.random.default_rng(seed)
    I0, I1 = band_image(dom, rng), band_image(dom, rng)
    v = smooth_flow(dom, rng, amp=amp, n_steps=cfg.n_time_steps, stationary=stationary,
                    gamma=cfg.gamma)
    w = smooth_flow(dom, rng, amp=amp, n_steps=cfg.n_time_steps, stationary=stationary,
                    gamma=cfg.gamma)
    out = dict(I0=I0, I1=I1, v=v.values, w=w.values, n_steps=cfg.n_time_steps,
               stationary=stationary, sigma2=cfg.sigma2, gamma=cfg.gamma, interp=cfg.interp,
               image_grad=cfg.image_grad, quadrature=cfg.quadrature,
               contraction=cfg.contraction)
    for tag, cls in (("state", StateObjective), ("def", DeformationObjective)):
        obj = cls(dom, I0, I1, cfg)
        t0 = time.perf_counter()
        ev = obj.gradient(v)
        out[f"{tag}_energy"] = obj.energy(v)
        out[f"{tag}_grad"] = ev.gradient.values
        out[f"{tag}_grad_energy"] = ev.energy
        out[f"{tag}_reg_energy"] = ev.reg_energy
        out[f"{tag}_data_energy"] = ev.data_energy
        out[f"{tag}_substeps"] = ev.cache.substeps
        out[f"{tag}_hvp_gn"] = ev.hessian_vector(w, gauss_newton=True).values
        out[f"{tag}_hvp_newton"] = ev.hessian_vector(w, gauss_newton=False).values
        out[f"{tag}_forward_end"] = ev.cache.forward[-1]
        print(f"  {name}/{tag}: {time.perf_counter() - t0:.1f}s")
    save(name, **dom_meta(dom), **out)


def solver_case(name):
    """Config 1 (tests/test_solver.py:122-127): 2-D 64², K=16, translation pair."""
    dom = Domain((64, 64), (16, 16), alpha=0.01, order=2)
    source, target, _ = synthesize_pair("translation", 64, shift=0.12)
    out = dict(source=source, target=target)
    for tag, cls in (("state", StateObjective), ("def", DeformationObjective)):
        obj = cls(dom, source, target, ProblemConfig(sigma2=0.03))
        cfg = SolverConfig(method="gauss_newton", max_outer=30, grad_tol=0.01)
        t0 = time.perf_counter()
        res = minimize(obj, TimeFlow.zero(dom), cfg)
        wall = time.perf_counter() - t0
        jd = gridops.jacobian_determinant(
            dom, spectral.include(dom, res.evaluation.cache.forward[-1], check=False))
        out[f"{tag}_status"] = res.status
        out[f"{tag}_energy"] = np.array([r.energy for r in res.records])
        out[f"{tag}_pcg"] = np.array([r.pcg_iters for r in res.records])
        out[f"{tag}_step"] = np.array([r.step for r in res.records])
        out[f"{tag}_negc"] = np.array([r.negative_curvature for r in res.records])
        out[f"{tag}_mse"] = np.array([r.mse_rel for r in res.records])
        out[f"{tag}_grel"] = np.array([r.grad_rel for r in res.records])
        out[f"{tag}_final_mse"] = res.final_mse_rel
        out[f"{tag}_final_grad_rel"] = res.final_grad_rel
        out[f"{tag}_final_energy"] = res.evaluation.energy
        out[f"{tag}_total_pcg"] = res.total_pcg_iters
        out[f"{tag}_jmin"], out[f"{tag}_jmax"] = float(jd.min()), float(jd.max())
        out[f"{tag}_velocity"] = res.velocity.values
        out[f"{tag}_wall_s"] = wall
        print(f"  {name}/{tag}: {res.status} {len(res.records)} records, {wall:.0f}s")
    save(name, **dom_meta(dom), **out)


def checksum_case(name, n, k):
    """§8(d) micro-benchmark recipe at 3-D n³: energy + GN HVP checksums."""
    dom = Domain((n,) * 3, (k,) * 3, alpha=0.02, order=2)
    rng = np.random.default_rng(0)
    I0, I1 = band_image(dom, rng), band_image(dom, rng)
    v = TimeFlow(dom, smooth_vector_block(dom, rng, 0.5 / n, decay=2.0)[None], 10, True)
    w = TimeFlow(dom, smooth_vector_block(dom, rng, 0.5 / n, decay=2.0)[None], 10, True)
    cfg = ProblemConfig(sigma2=0.1, n_time_steps=10)
    out = dict(n=n, k=k)
    for tag, cls in (("state", StateObjective), ("def", DeformationObjective)):
        obj = cls(dom, I0, I1, cfg)
        t0 = time.perf_counter()
        ev = obj.gradient(v)
        hw = ev.hessian_vector(w, gauss_newton=True).values
        out[f"{tag}_energy"] = ev.energy
        out[f"{tag}_grad_norm"] = np.linalg.norm(ev.gradient.values)
        out[f"{tag}_hvp_norm"] = np.linalg.norm(hw)
        out[f"{tag}_hvp_dot_w"] = spectral.inner(hw, w.values)
        out[f"{tag}_grad_dot_w"] = spectral.inner(ev.gradient.values, w.values)
        print(f"  {name}/{tag}: {time.perf_counter() - t0:.0f}s")
    save(name, **dom_meta(dom), **out)


N_SAMPLES = 1000


def _vector_summary(prefix, x, w, r, idx):
    """Full-precision fingerprint of one band vector (a few KB, not 13 MB):
    Frobenius norm, Re<x, w>, Re<x, r> against a seeded probe, and the complex
    coefficients at ``idx`` (flat indices into ``x``)."""
    return {f"{prefix}_norm": np.linalg.norm(x), f"{prefix}_dot_w": spectral.inner(x, w),
            f"{prefix}_dot_r": spectral.inner(x, r), f"{prefix}_samples": x.reshape(-1)[idx]}


def headline_probe(shape):
    """Seeded probe vector and sample indices shared by the generator and the
    GPU test (plain numpy, so the GPU box regenerates them bit-identically)."""
    rng = np.random.default_rng(20260)
    r = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    idx = np.sort(rng.choice(int(np.prod(shape)), N_SAMPLES, replace=False))
    return r, idx


def headline_case(tag):
    """BASELINE config 3 at full precision: 128³/K=32,
    Nt=10, the §8(d) micro-benchmark recipe, one objective per process
    (~20 CPU-minutes each).  Energy, gradient, GN and Newton HVP."""
    n, k = 128, 32
    dom = Domain((n,) * 3, (k,) * 3, alpha=0.02, order=2)
    rng = np.random.default_rng(0)
    I0, I1 = band_image(dom, rng), band_image(dom, rng)
    v = TimeFlow(dom, smooth_vector_block(dom, rng, 0.5 / n, decay=2.0)[None], 10, True)
    w = TimeFlow(dom, smooth_vector_block(dom, rng, 0.5 / n, decay=2.0)[None], 10, True)
    cfg = ProblemConfig(sigma2=0.1, n_time_steps=10)
    cls = {"state": StateObjective, "def": DeformationObjective}[tag]
    r, idx = headline_probe(v.values.shape)
    obj = cls(dom, I0, I1, cfg)
    out = dict(n=n, k=k, sample_idx=idx)
    t0 = time.perf_counter()
    out["energy_direct"] = obj.energy(v)
    ev = obj.gradient(v)
    out["energy"], out["reg_energy"], out["data_energy"] = ev.energy, ev.reg_energy, ev.data_energy
    out["substeps"] = ev.cache.substeps
    out.update(_vector_summary("grad", ev.gradient.values, w.values, r, idx))
    out["t_grad_s"] = time.perf_counter() - t0
    for gn, name in ((True, "hvp_gn"), (False, "hvp_newton")):
        t0 = time.perf_counter()
        hw = ev.hessian_vector(w, gauss_newton=gn).values
        out[f"t_{name}_s"] = time.perf_counter() - t0
        out.update(_vector_summary(name, hw, w.values, r, idx))
        print(f"  headline_128/{tag}/{name}: {out[f't_{name}_s']:.0f}s", flush=True)
    save(f"headline_128_{tag}", **dom_meta(dom), **out)


def blob_pair_ref(dom, seed=1):
    """Seeded 3-D pair (the bench's ``blob_pair`` recipe) built with the
    reference's own helpers: six periodic bumps; target = cubic warp of the
    source by a band-4 smooth displacement of ~3 voxels."""
    n = dom.shape[0]
    rng = np.random.default_rng(seed)
    axes = [np.arange(s) / s for s in dom.shape]
    mesh = np.meshgrid(*axes, indexing="ij")
    src = np.zeros(dom.shape)
    for _ in range(6):
        c = 0.3 + 0.4 * rng.random(3)
        sharp = 8.0 + 16.0 * rng.random()
        b = np.ones(dom.shape)
        for x, cc in zip(mesh, c):
            b = b * np.exp(sharp * (np.cos(2 * np.pi * (x - cc)) - 1.0))
        src += (0.5 + 0.5 * rng.random()) * b
    src /= src.max()
    ddom = Domain(dom.shape, (4,) * dom.ndim)
    disp = spectral.include(ddom, smooth_vector_block(ddom, rng, 3.0 / n, decay=2.0))
    return src, gridops.warp(ddom, src, disp, interp="cubic")


def config2_case(tag):
    """SURVEY config 2 end to end: 3-D 64³/K=16 blob pair,
    alpha=0.01, s=2, sigma²=0.03, ``SolverConfig()`` defaults, one objective
    per process."""
    dom = Domain((64,) * 3, (16,) * 3, alpha=0.01, order=2)
    source, target = blob_pair_ref(dom)
    cls = {"state": StateObjective, "def": DeformationObjective}[tag]
    obj = cls(dom, source, target, ProblemConfig(sigma2=0.03))
    t0 = time.perf_counter()
    res = minimize(obj, TimeFlow.zero(dom), SolverConfig())
    wall = time.perf_counter() - t0
    jd = gridops.jacobian_determinant(
        dom, spectral.include(dom, res.evaluation.cache.forward[-1], check=False))
    r, idx = headline_probe(res.velocity.values.shape)
    out = dict(source=source, target=target, status=res.status,
               energy=np.array([x.energy for x in res.records]),
               pcg=np.array([x.pcg_iters for x in res.records]),
               step=np.array([x.step for x in res.records]),
               negc=np.array([x.negative_curvature for x in res.records]),
               mse=np.array([x.mse_rel for x in res.records]),
               grel=np.array([x.grad_rel for x in res.records]),
               final_mse=res.final_mse_rel, final_grad_rel=res.final_grad_rel,
               final_energy=res.evaluation.energy, total_pcg=res.total_pcg_iters,
               jmin=float(jd.min()), jmax=float(jd.max()), wall_s=wall,
               sample_idx=idx, velocity_norm=np.linalg.norm(res.velocity.values),
               velocity_samples=res.velocity.values.reshape(-1)[idx])
    print(f"  config2_64/{tag}: {res.status} {len(res.records)} records, {wall:.0f}s", flush=True)
    save(f"config2_64_{tag}", **dom_meta(dom), **out)


def volio_case(name):
    """BLVOL files written by the reference writer (volio.py), stored as bytes."""
    import tempfile

    from blreg import volio

    rng = np.random.default_rng(21)
    scalar = rng.standard_normal((5, 6, 7))
    vector = rng.standard_normal((2, 9, 4))
    out = dict(scalar=scalar, vector=vector)
    with tempfile.TemporaryDirectory() as tmp:
        for tag, arr, spacing in (("scalar", scalar, None), ("vector", vector, (0.5, 0.25))):
            path = os.path.join(tmp, f"{tag}.vol")
            volio.write_volume(path, arr, spacing)
            with open(path, "rb") as fh:
                out[f"{tag}_bytes"] = np.frombuffer(fh.read(), dtype=np.uint8)
    save(name, **out)


def main():
    if "--headline" in sys.argv:  # --headline state|def (one objective per process)
        headline_case(sys.argv[sys.argv.index("--headline") + 1])
        return
    if "--config2" in sys.argv:  # --config2 state|def
        config2_case(sys.argv[sys.argv.index("--config2") + 1])
        return
    slow = "--slow" in sys.argv
    spectral_case("spectral_3d", Domain((12, 16, 18), (3, 4, 5), alpha=0.05), 1)
    spectral_case("spectral_2d", Domain((32, 30), (8, 7), alpha=0.05), 2)
    spectral_case("spectral_1d", Domain((32,), (8,), alpha=0.05), 3)
    spectral_case("spectral_nyq", Domain((8, 12), (4, 6), alpha=0.05), 4)
    rhs_case("rhs_3d", Domain((12, 16, 18), (3, 4, 5), alpha=0.05), 5)
    rhs_case("rhs_2d", Domain((32, 32), (8, 8), alpha=0.05), 6)
    transport_case("transport_3d", Domain((16, 16, 16), (4, 4, 4)), 7, 6, 1, True)
    transport_case("transport_3d_sub", Domain((12, 16, 18), (3, 4, 5)), 8, 4, 2, True)
    transport_case("transport_2d_ns", Domain((32, 32), (8, 8)), 9, 6, 1, False)
    grid_case("grid_3d", Domain((12, 16, 18), (3, 4, 5)), 10)
    grid_case("grid_2d", Domain((32, 30), (8, 7)), 11)
    d3 = Domain((16, 16, 16), (4, 4, 4), alpha=0.05)
    objective_case("obj_3d", d3, 12, ProblemConfig(sigma2=0.1, n_time_steps=6))
    objective_case("obj_3d_cubic_gamma", d3, 13,
                   ProblemConfig(sigma2=0.1, n_time_steps=6, gamma=1, interp="cubic",
                                 quadrature="simpson"))
    objective_case("obj_3d_direct_spec", d3, 14,
                   ProblemConfig(sigma2=0.1, n_time_steps=6, contraction="direct",
                                 image_grad="spectral"))
    objective_case("obj_2d", Domain((32, 32), (8, 8), alpha=0.05), 15,
                   ProblemConfig(sigma2=0.1, n_time_steps=10))
    objective_case("obj_2d_ns", Domain((32, 32), (8, 8), alpha=0.05), 16,
                   ProblemConfig(sigma2=0.1, n_time_steps=6), stationary=False)
    objective_case("obj_2d_refine", Domain((32, 32), (8, 8), alpha=0.05), 17,
                   ProblemConfig(sigma2=0.1, n_time_steps=4), amp=0.3)
    volio_case("volio")
    if slow:
        solver_case("solver_config1")
        checksum_case("checksum_64", 64, 16)


if __name__ == "__main__":
    main()
