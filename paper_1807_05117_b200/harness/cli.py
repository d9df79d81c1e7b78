"""``python -m paper_1807_05117_b200.harness.cli`` — the CLI the reference
declares (``pyproject.toml:20``, ``SPEC.md:514``): ``register``,
``synthesize``, ``check-derivatives``, ``report``.

Exit codes ("category codes"): 0 success, 2 configuration error,
3 input error, 4 CFL violation (auto-refine off), 5 solver stalled or out of
budget, 6 derivative check failed.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

EXIT_OK, EXIT_CONFIG, EXIT_INPUT, EXIT_CFL, EXIT_STALL, EXIT_CHECK = 0, 2, 3, 4, 5, 6


def _periodic_blobs(shape, rng, n=6, sharp=(8.0, 24.0)):
    """Sum of n periodic bumps exp(s (cos 2 pi (x - c) - 1)), s in ``sharp``."""
    axes = [np.arange(s) / s for s in shape]
    mesh = np.meshgrid(*axes, indexing="ij")
    img = np.zeros(shape)
    for _ in range(n):
        c = 0.3 + 0.4 * rng.random(len(shape))
        sharp_k = sharp[0] + (sharp[1] - sharp[0]) * rng.random()
        b = np.ones(shape)
        for x, cc in zip(mesh, c):
            b = b * np.exp(sharp_k * (np.cos(2 * np.pi * (x - cc)) - 1.0))
        img += (0.5 + 0.5 * rng.random()) * b
    return img / img.max()


def synthesize(kind: str, size: int, ndim: int, seed: int, shift: float = 0.1, amp: float = 3.0):
    """Deterministic periodic pairs on the B200 path.  ``blobs``: bumps, target
    = cubic warp of the source by a band-4 smooth displacement of ~``amp``
    voxels; ``translation``: target = source shifted by ``shift`` of the box
    along the first axis (exact Fourier shift).  Returns (source, target)."""
    import torch

    from .. import Domain, gridops, spectral
    from ..spectral import as_band

    shape = (size,) * ndim
    rng = np.random.default_rng(seed)
    # translation: three broad bumps (resolved at any grid size); blobs: six sharper ones
    src = _periodic_blobs(shape, rng, 3, (2.0, 6.0)) if kind == "translation" else _periodic_blobs(shape, rng)
    dom = Domain(shape, (4,) * ndim)
    if kind == "translation":
        disp = torch.zeros((ndim,) + shape, dtype=torch.float64, device=dom.torch_device)
        disp[0] = -shift
        tgt = gridops.fourier_warp(dom, torch.from_numpy(src), disp)
    elif kind == "blobs":
        c = rng.standard_normal((ndim,) + dom.block_shape) + 1j * rng.standard_normal((ndim,) + dom.block_shape)
        c = spectral.symmetrize(dom, as_band(dom, c))
        k2 = sum(np.meshgrid(*[np.fft.fftfreq(m, 1.0 / m) ** 2 for m in dom.block_shape], indexing="ij"))
        c = c / torch.from_numpy((1.0 + k2) ** 2.0).to(c.device)
        c = c * (amp / size / spectral.max_abs(dom, c))
        tgt = gridops.warp(dom, torch.from_numpy(src), spectral.include(dom, c), "cubic")
    else:
        raise ValueError(f"unknown kind {kind!r} (blobs, translation)")
    return src, tgt.double().cpu().numpy()


def cmd_synthesize(args) -> int:
    from ..outputs import write_volume

    src, tgt = synthesize(args.kind, args.size, args.ndim, args.seed, args.shift, args.amp)
    os.makedirs(args.out, exist_ok=True)
    write_volume(os.path.join(args.out, "source.vol"), src)
    write_volume(os.path.join(args.out, "target.vol"), tgt)
    print(f"wrote {args.out}/source.vol, {args.out}/target.vol ({args.kind}, {src.shape})")
    return EXIT_OK


def cmd_register(args) -> int:
    from .. import DeformationObjective, StateObjective, TimeFlow, gridops, minimize, spectral
    from ..outputs import read_volume, write_volume
    from ..transport import CFLViolation
    from . import report as R
    from .runconfig import ConfigError, effective_settings, load_config

    try:
        cfg = load_config(args.config)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    base = os.path.dirname(os.path.abspath(args.config))
    try:
        src, _ = read_volume(os.path.join(base, cfg.source))
        tgt, _ = read_volume(os.path.join(base, cfg.target))
        if src.shape != tgt.shape:
            raise ValueError(f"source {src.shape} and target {tgt.shape} grids differ")
        dom = cfg.domain_for(src.shape)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except (OSError, ValueError) as e:
        print(f"input error: {e}", file=sys.stderr)
        return EXIT_INPUT
    cls = DeformationObjective if cfg.objective == "deformation" else StateObjective
    obj = cls(dom, src.astype(np.float64), tgt.astype(np.float64), cfg.problem)
    v0 = TimeFlow.zero(dom, cfg.problem.n_time_steps, cfg.mode == "stationary")
    t0 = time.perf_counter()
    try:
        res = minimize(obj, v0, cfg.solver)
    except CFLViolation as e:
        print(f"CFL violation: {e}", file=sys.stderr)
        return EXIT_CFL
    wall = time.perf_counter() - t0
    disp = spectral.include(dom, res.evaluation.cache.forward[-1], check=False)
    jd = gridops.jacobian_determinant(dom, disp)
    warped = res.evaluation.warped_source
    out = os.path.join(base, cfg.output_dir) if not os.path.isabs(cfg.output_dir) else cfg.output_dir
    os.makedirs(out, exist_ok=True)
    write_volume(os.path.join(out, "warped.vol"), warped)
    write_volume(os.path.join(out, "displacement.vol"), disp)
    write_volume(os.path.join(out, "difference.vol"), warped - obj.target_d)
    R.write_csv(res.records, os.path.join(out, "iterations.csv"))
    rep = R.RegistrationReport(records=res.records, status=res.status, final_mse_rel=float(res.final_mse_rel),
                               final_grad_rel=float(res.final_grad_rel), jacobian_min=float(jd.min()),
                               jacobian_max=float(jd.max()), settings=effective_settings(cfg, dom),
                               total_time=wall, negative_curvature_events=res.negative_curvature_events,
                               total_pcg_iters=res.total_pcg_iters)
    R.write_report(rep, os.path.join(out, "report.txt"))
    print(R.report_text(rep))
    return EXIT_OK if res.status == "converged" else EXIT_STALL


def fd_checks(size: int, ndim: int, seed: int, eps: float = 1e-4) -> list:
    """Gradient and Newton-HVP central-difference checks and the GN curvature
    bound for both objectives (SPEC harness check_derivatives), N <= 64."""
    from .. import DeformationObjective, Domain, ProblemConfig, StateObjective, TimeFlow
    from ..spectral import as_band
    from ..transport import flow_inner

    if size > 64:
        raise ValueError("check-derivatives is limited to N <= 64")
    shape = (size,) * ndim
    dom = Domain(shape, (size // 4,) * ndim, alpha=0.05)
    rng = np.random.default_rng(seed)

    def band_image():  # band-limited to the domain's band (the reference tests' band_image recipe)
        import torch

        from .. import spectral

        c = rng.standard_normal(dom.block_shape) + 1j * rng.standard_normal(dom.block_shape)
        c = spectral.symmetrize(dom, as_band(dom, c))
        k2 = sum(np.meshgrid(*[np.fft.fftfreq(m, 1.0 / m) ** 2 for m in dom.block_shape], indexing="ij"))
        img = spectral.include(dom, c / torch.from_numpy((1.0 + k2) ** 3.0).to(c.device))
        img = img - img.min()
        return (img / img.max()).cpu().numpy()

    src, tgt = band_image(), band_image()

    def flow(amp):
        import torch

        from .. import spectral

        c = rng.standard_normal((ndim,) + dom.block_shape) + 1j * rng.standard_normal((ndim,) + dom.block_shape)
        c = spectral.symmetrize(dom, as_band(dom, c))
        k2 = sum(np.meshgrid(*[np.fft.fftfreq(m, 1.0 / m) ** 2 for m in dom.block_shape], indexing="ij"))
        c = c / torch.from_numpy((1.0 + k2) ** 3.0).to(c.device)
        c = c * (amp / spectral.max_abs(dom, c))
        return TimeFlow(dom, c[None], 32, True)

    # the reference probe's discretization (probe_hvp.py setup: Nt = 32, Fourier
    # interpolation, spectral image gradients, Simpson quadrature)
    cfg = ProblemConfig(sigma2=1.0, n_time_steps=32, interp="fourier", image_grad="spectral",
                        quadrature="simpson")
    rows = []
    for cls in (StateObjective, DeformationObjective):
        obj = cls(dom, src, tgt, cfg)
        v, w = flow(0.04), flow(0.04)
        ev = obj.gradient(v)
        pred = flow_inner(ev.gradient, w, cfg.quadrature)
        fd = (obj.energy(v + eps * w) - obj.energy(v - eps * w)) / (2 * eps)
        rows.append((cls.__name__, "gradient FD", abs(pred - fd) / abs(fd), 1e-6))
        hv = ev.hessian_vector(w, gauss_newton=False)
        d = (obj.gradient(v + eps * w).gradient - obj.gradient(v - eps * w).gradient) * (1.0 / (2 * eps))
        err = np.sqrt(flow_inner(hv - d, hv - d, cfg.quadrature) / flow_inner(hv, hv, cfg.quadrature))
        rows.append((cls.__name__, "Newton HVP FD", err, 1e-4))
        worst = np.inf
        for _ in range(5):
            u = flow(1.0)
            q = flow_inner(ev.hessian_vector(u, gauss_newton=True), u, cfg.quadrature)
            from .. import spectral

            lu = u.map_nodes(lambda c: spectral.apply_helmholtz(dom, c))
            ref = flow_inner(lu, u, cfg.quadrature)
            worst = min(worst, (q - ref) / ref)
        rows.append((cls.__name__, "GN curvature margin", -worst if worst < 0 else 0.0, 1e-8))
    return rows


def cmd_check(args) -> int:
    rows = fd_checks(args.size, args.ndim, args.seed)
    ok = True
    print(f"{'objective':22s} {'check':22s} {'rel. error':>12s} {'bound':>8s}")
    for name, check, err, bound in rows:
        good = err <= bound
        ok = ok and good
        print(f"{name:22s} {check:22s} {err:12.3e} {bound:8.0e} {'ok' if good else 'FAIL'}")
    return EXIT_OK if ok else EXIT_CHECK


def cmd_report(args) -> int:
    from . import report as R

    path = args.path
    if os.path.isdir(path):
        path = os.path.join(path, "report.json")
    try:
        with open(path) as fh:
            rep = R.RegistrationReport.from_json(fh.read())
    except (OSError, ValueError, KeyError) as e:
        print(f"input error: {e}", file=sys.stderr)
        return EXIT_INPUT
    sys.stdout.write(R.report_text(rep))
    if args.csv:
        sys.stdout.write(R.records_to_csv(rep.records))
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="blreg-b200", description=__doc__.splitlines()[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("register", help="run a registration from an INI config")
    p.add_argument("config")
    p.set_defaults(fn=cmd_register)
    p = sub.add_parser("synthesize", help="write a deterministic synthetic pair (BLVOL)")
    p.add_argument("kind", choices=["blobs", "translation"])
    p.add_argument("--size", type=int, default=64)
    p.add_argument("--ndim", type=int, default=3)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--shift", type=float, default=0.1)
    p.add_argument("--amp", type=float, default=3.0)
    p.add_argument("--out", default="pair")
    p.set_defaults(fn=cmd_synthesize)
    p = sub.add_parser("check-derivatives", help="finite-difference gradient / HVP checks")
    p.add_argument("--size", type=int, default=32)
    p.add_argument("--ndim", type=int, default=2)
    p.add_argument("--seed", type=int, default=0)
    p.set_defaults(fn=cmd_check)
    p = sub.add_parser("report", help="print a saved registration report")
    p.add_argument("path", help="run output directory or report.json")
    p.add_argument("--csv", action="store_true")
    p.set_defaults(fn=cmd_report)
    args = ap.parse_args(argv)
    return args.fn(args)


if __name__ == "__main__":
    sys.exit(main())
