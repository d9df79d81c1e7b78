"""Operations on real fields sampled on the full grid (mirrors ``blreg/gridops.py``).

Periodic warps (nearest / trilinear / cubic B-spline), central and spectral
gradients and the Jacobian determinant run in the sm_100a library.  The exact
trigonometric ``fourier`` warp is a verification-only operator in the
reference (O(N^(d+1)) memory, ``gridops.py:51-75``); here it is evaluated with
dense device matmuls for the same small verification problems.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .domain import Domain
from .spectral import as_grid, ptr

_INTERP = {"nearest": 0, "linear": 1, "cubic": 3}


def interp_code(interp: str) -> int:
    code = _INTERP.get(interp)
    if code is None:
        raise ValueError(f"unknown interpolation {interp!r}")
    return code


def warp(domain: Domain, values, displacement, interp: str = "linear") -> torch.Tensor:
    """Evaluate ``values`` at ``x + u(x)``, periodically (gridops.py:32-48)."""
    if interp == "fourier":
        return fourier_warp(domain, values, displacement)
    f = as_grid(domain, values)
    u = as_grid(domain, displacement)
    nimg = f.numel() // domain.n_grid
    out = torch.empty_like(f)
    _lib.call("blr_warp", domain.ctx().bind(), ptr(f), nimg, ptr(u), 1, interp_code(interp), ptr(out))
    return out


def warp_nodes(domain: Domain, values, displacements, interp: str = "linear") -> torch.Tensor:
    """One image warped by a stack of displacements ``(n, d, *shape)`` in one launch."""
    if interp == "fourier":
        return torch.stack([fourier_warp(domain, values, u) for u in displacements])
    f = as_grid(domain, values)
    u = as_grid(domain, displacements)
    n = u.shape[0]
    out = torch.empty((n,) + domain.shape, dtype=domain.rdtype, device=domain.torch_device)
    _lib.call("blr_warp", domain.ctx().bind(), ptr(f), 1, ptr(u), n, interp_code(interp), ptr(out))
    return out


def fourier_warp(domain: Domain, values, displacement) -> torch.Tensor:
    """Trigonometric interpolant at ``x + u(x)`` (gridops.py:51-75), verification only."""
    shape, d = domain.shape, domain.ndim
    f = as_grid(domain, values).double()
    if f.dim() > d:  # stack of images sharing one displacement
        flat = f.reshape((-1,) + shape)
        return torch.stack([fourier_warp(domain, x, displacement) for x in flat]).reshape(f.shape).to(
            domain.rdtype)
    u = as_grid(domain, displacement).double()
    spec = torch.fft.fftn(f) / float(np.prod(shape))
    npts = int(np.prod(shape))
    phases = []
    for ax, n in enumerate(shape):
        idx = torch.arange(n, dtype=torch.float64, device=f.device).reshape(
            [n if a == ax else 1 for a in range(d)])
        x = ((idx + u[ax] * n) / n).reshape(npts)
        fr = torch.from_numpy(np.rint(np.fft.fftfreq(n, 1.0 / n))).to(f.device)
        ph = torch.exp(2j * np.pi * torch.outer(x, fr))
        if n % 2 == 0:
            ph[:, n // 2] = torch.cos(2.0 * np.pi * x * (n // 2))
        phases.append(ph)
    acc = torch.tensordot(spec, phases[-1], dims=([d - 1], [1]))
    for ax in range(d - 2, -1, -1):
        acc = torch.einsum("...kp,pk->...p", acc, phases[ax])
    return acc.real.reshape(shape).to(domain.rdtype).contiguous()


def spatial_gradient(domain: Domain, values, mode: str = "central") -> torch.Tensor:
    """Gradient of scalar grid field(s) (gridops.py:78-100); leading dims batch."""
    f = as_grid(domain, values)
    lead = tuple(f.shape[:-domain.ndim])
    nf = int(np.prod(lead)) if lead else 1
    if mode not in ("central", "spectral"):
        raise ValueError(f"unknown gradient mode {mode!r}")
    out = torch.empty(lead + (domain.ndim,) + domain.shape, dtype=domain.rdtype,
                      device=domain.torch_device)
    _lib.call("blr_grid_gradient", domain.ctx().bind(), ptr(f), nf, 0 if mode == "central" else 1,
              ptr(out))
    return out


def jacobian_matrix(domain: Domain, displacement) -> torch.Tensor:
    d = domain.ndim
    g = spatial_gradient(domain, displacement)  # (d, d, *shape): g[i, j] = d_j u_i
    eye = torch.eye(d, dtype=domain.rdtype, device=domain.torch_device).reshape((d, d) + (1,) * d)
    return g + eye


def jacobian_determinant(domain: Domain, displacement) -> torch.Tensor:
    """det(I + Du) by central differences (gridops.py:103-131)."""
    u = as_grid(domain, displacement)
    out = torch.empty(domain.shape, dtype=domain.rdtype, device=domain.torch_device)
    _lib.call("blr_jacobian_det", domain.ctx().bind(), ptr(u), ptr(out))
    return out
