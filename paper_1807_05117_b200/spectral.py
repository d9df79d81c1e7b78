"""Band-limited spectral algebra on the B200 (mirrors ``blreg/spectral.py``).

Coefficient blocks are CUDA tensors (complex128 / complex64) in FFT wrap
order with the reference's shapes: scalar ``block_shape``, vector
``(d, *block_shape)``, matrix ``(d, d, *block_shape)``.  Grid fields are real
CUDA tensors.  numpy inputs are accepted and copied to the device once.
Every numeric operation runs in the sm_100a library (``include/blreg_b200.h``).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .domain import Domain

_TWO_PI = 2.0 * np.pi


# ---------------------------------------------------------------------------
# tensor plumbing
# ---------------------------------------------------------------------------

def as_band(domain: Domain, x) -> torch.Tensor:
    """Contiguous device tensor of the domain's complex dtype."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=domain.torch_device, dtype=domain.cdtype)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).to(
            device=domain.torch_device, dtype=domain.cdtype)
    return t.contiguous()


def as_grid(domain: Domain, x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(device=domain.torch_device, dtype=domain.rdtype)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(
            device=domain.torch_device, dtype=domain.rdtype)
    return t.contiguous()


def ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def to_numpy(t):
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def _grid_id(domain: Domain, grid_shape) -> int:
    if grid_shape is None or tuple(grid_shape) == domain.shape:
        return 0
    if tuple(grid_shape) == domain.pad:
        return 1
    raise ValueError(f"grid_shape must be the image grid {domain.shape} or the pad grid {domain.pad}")


def _nlead(x: torch.Tensor, d: int) -> tuple:
    return tuple(x.shape[:-d])


# ---------------------------------------------------------------------------
# symmetry (spectral.py:37-56)
# ---------------------------------------------------------------------------

def symmetrize(domain: Domain, coeffs) -> torch.Tensor:
    c = as_band(domain, coeffs)
    out = torch.empty_like(c)
    nb = int(np.prod(c.shape[:-domain.ndim])) if c.dim() > domain.ndim else 1
    _lib.call("blr_symmetrize", domain.ctx().bind(), ptr(c), nb, ptr(out))
    return out


def symmetry_error(domain: Domain, coeffs) -> float:
    c = as_band(domain, coeffs)
    scale = float(c.abs().max()) if c.numel() else 0.0
    if scale == 0.0:
        return 0.0
    s = symmetrize(domain, c)
    return float((2.0 * (c - s)).abs().max()) / scale


# ---------------------------------------------------------------------------
# include / project (spectral.py:89-153)
# ---------------------------------------------------------------------------

def include(domain: Domain, coeffs, grid_shape=None, check: bool = True, deriv=None) -> torch.Tensor:
    """Realize band blocks as real fields on the image grid or the pad grid.

    ``deriv`` (optional, one entry per realized field): component axis ``j``
    realizes ``d_j`` of the field (``spectral_gradient`` fused), -1 none.
    Raises ``ValueError`` when the symmetry violation exceeds 1e-10
    (``spectral.py:104-105``).
    """
    d = domain.ndim
    c = as_band(domain, coeffs)
    if tuple(c.shape[-d:]) != domain.block_shape:
        raise ValueError(f"block shape {tuple(c.shape[-d:])} does not match domain {domain.block_shape}")
    if check and symmetry_error(domain, c) > 1e-10:
        raise ValueError("coefficients violate conjugate symmetry; spectrum is corrupted")
    gid = _grid_id(domain, grid_shape)
    grid = domain.shape if gid == 0 else domain.pad
    lead = _nlead(c, d)
    nf = int(np.prod(lead)) if lead else 1
    out = torch.empty(lead + grid, dtype=domain.rdtype, device=domain.torch_device)
    dv = None
    if deriv is not None:
        deriv = list(deriv)
        if len(deriv) != nf:
            raise ValueError("deriv needs one entry per field")
        dv = _lib.int_array(deriv)
    _lib.call("blr_include", domain.ctx().bind(), gid, ptr(c), nf, dv, ptr(out))
    return out


def project(domain: Domain, values, grid_shape=None) -> torch.Tensor:
    """Band-limit real fields: forward DFT, truncate, symmetrize (spectral.py:122-135)."""
    d = domain.ndim
    f = as_grid(domain, values)
    gid = _grid_id(domain, grid_shape)
    grid = domain.shape if gid == 0 else domain.pad
    if tuple(f.shape[-d:]) != tuple(grid):
        raise ValueError(f"field shape {tuple(f.shape[-d:])} does not match grid {grid}")
    lead = _nlead(f, d)
    nf = int(np.prod(lead)) if lead else 1
    out = torch.empty(lead + domain.block_shape, dtype=domain.cdtype, device=domain.torch_device)
    _lib.call("blr_project", domain.ctx().bind(), gid, ptr(f), nf, ptr(out))
    return out


def _pad_shape(domain: Domain) -> tuple:
    return domain.pad


def _to_pad_grid(domain: Domain, coeffs) -> torch.Tensor:
    return include(domain, coeffs, domain.pad, check=False)


def _from_pad_grid(domain: Domain, values) -> torch.Tensor:
    return project(domain, values, domain.pad)


# ---------------------------------------------------------------------------
# truncated convolution (spectral.py:156-217)
# ---------------------------------------------------------------------------

def conv_matvec(domain: Domain, mat, vec, transpose: bool = False) -> torch.Tensor:
    """``sum_j M[i, j] * v[j]`` (or the transpose), band-limited."""
    M, v = as_band(domain, mat), as_band(domain, vec)
    out = torch.empty_like(v)
    _lib.call("blr_conv_matvec", domain.ctx().bind(), ptr(M), ptr(v), int(bool(transpose)), ptr(out))
    return out


def conv_scalar(domain: Domain, a, b) -> torch.Tensor:
    ag, bg = _to_pad_grid(domain, a), _to_pad_grid(domain, b)
    prod = torch.empty_like(ag)
    _lib.call("blr_mul", domain.ctx().bind(), ptr(ag), ptr(bg), ag.numel(), ptr(prod))
    return _from_pad_grid(domain, prod)


def conv_dot(domain: Domain, a, b) -> torch.Tensor:
    ag, bg = _to_pad_grid(domain, a), _to_pad_grid(domain, b)
    return _from_pad_grid(domain, (ag * bg).sum(0))


def truncated_convolution(domain: Domain, a, b) -> torch.Tensor:
    """Dispatch on operand rank (spectral.py:156-178)."""
    d = domain.ndim
    ra, rb = a.ndim - d, b.ndim - d
    if ra == 0 and rb == 0:
        return conv_scalar(domain, a, b)
    if ra == 2 and rb == 1:
        return conv_matvec(domain, a, b)
    if ra == 1 and rb == 0:
        return _from_pad_grid(domain, _to_pad_grid(domain, a) * _to_pad_grid(domain, b)[None])
    if ra == 0 and rb == 1:
        return truncated_convolution(domain, b, a)
    if ra == 1 and rb == 1:
        return conv_dot(domain, a, b)
    raise ValueError(f"unsupported operand ranks ({ra}, {rb})")


# ---------------------------------------------------------------------------
# diagonal operators (spectral.py:242-328)
# ---------------------------------------------------------------------------

def _angular_frequencies(domain: Domain):
    d = domain.ndim
    out = []
    for ax, f in enumerate(domain.frequencies()):
        shape = [1] * d
        shape[ax] = f.size
        out.append(_TWO_PI * f.astype(np.float64).reshape(shape))
    return tuple(out)


def metric_symbol(domain: Domain) -> np.ndarray:
    """Host copy of ``A(k)**order`` (spectral.py:260-262)."""
    acc = np.zeros(domain.block_shape, dtype=np.float64)
    for ax, (f, n) in enumerate(zip(domain.frequencies(), domain.shape)):
        shape = [1] * domain.ndim
        shape[ax] = f.size
        if domain.symbol == "discrete":
            term = 2.0 * n * n * (1.0 - np.cos(_TWO_PI * f / n))
        else:
            term = (_TWO_PI * f) ** 2
        acc = acc + term.reshape(shape)
    return (1.0 + domain.alpha * acc) ** domain.order


def _nblocks(domain: Domain, c: torch.Tensor) -> int:
    lead = c.shape[:-domain.ndim]
    return int(np.prod(lead)) if len(lead) else 1


def apply_helmholtz(domain: Domain, coeffs) -> torch.Tensor:
    c = as_band(domain, coeffs)
    out = torch.empty_like(c)
    _lib.call("blr_helmholtz", domain.ctx().bind(), ptr(c), _nblocks(domain, c), 0, ptr(out))
    return out


def apply_inverse_helmholtz(domain: Domain, coeffs) -> torch.Tensor:
    c = as_band(domain, coeffs)
    out = torch.empty_like(c)
    _lib.call("blr_helmholtz", domain.ctx().bind(), ptr(c), _nblocks(domain, c), 1, ptr(out))
    return out


def _ik(domain: Domain, ax: int) -> torch.Tensor:
    k = _angular_frequencies(domain)[ax]
    return torch.from_numpy(1j * k).to(device=domain.torch_device, dtype=domain.cdtype)


def spectral_gradient(domain: Domain, scalar) -> torch.Tensor:
    s = as_band(domain, scalar)
    return torch.stack([_ik(domain, ax) * s for ax in range(domain.ndim)])


def spectral_divergence(domain: Domain, vec) -> torch.Tensor:
    v = as_band(domain, vec)
    out = torch.empty(v.shape[1:], dtype=domain.cdtype, device=domain.torch_device)
    _lib.call("blr_divergence", domain.ctx().bind(), ptr(v), 1, ptr(out))
    return out


def spectral_jacobian(domain: Domain, vec) -> torch.Tensor:
    v = as_band(domain, vec)
    d = domain.ndim
    return torch.stack([torch.stack([_ik(domain, j) * v[i] for j in range(d)]) for i in range(d)])


def leray_projection(domain: Domain, vec):
    v = as_band(domain, vec)
    w = make_divergence_free(domain, v)
    div = spectral_divergence(domain, v)
    lap = torch.from_numpy(sum(-(k ** 2) for k in _angular_frequencies(domain))).to(
        device=domain.torch_device, dtype=domain.rdtype)
    p = torch.where(lap != 0, div / torch.where(lap != 0, lap, torch.ones_like(lap)),
                    torch.zeros_like(div))
    return w, p


def make_divergence_free(domain: Domain, vec) -> torch.Tensor:
    v = as_band(domain, vec)
    out = torch.empty_like(v)
    nvec = int(np.prod(v.shape[:-domain.ndim - 1])) if v.dim() > domain.ndim + 1 else 1
    _lib.call("blr_leray", domain.ctx().bind(), ptr(v), nvec, ptr(out))
    return out


# ---------------------------------------------------------------------------
# inner products and norms (spectral.py:335-350)
# ---------------------------------------------------------------------------

def inner(a, b, domain: Domain | None = None) -> float:
    """``Re sum a * conj(b)`` over all coefficients (deterministic reduction)."""
    if domain is None:
        domain = _domain_of(a)
    ta, tb = as_band(domain, a), as_band(domain, b)
    if ta.shape != tb.shape:
        raise ValueError("inner product of differently shaped blocks")
    res = _lib.out_double()
    _lib.call("blr_inner", domain.ctx().bind(), ptr(ta), ptr(tb), ta.numel(), C.byref(res))
    return float(res.value)


def grid_inner(domain: Domain, f, g) -> float:
    tf, tg = as_grid(domain, f), as_grid(domain, g)
    return domain.cell_volume * float((tf.double() * tg.double()).sum())


def grid_norm2(domain: Domain, f, g=None) -> float:
    """``cell_volume * sum f^2`` (or of ``f - g``), reduced on the device."""
    tf = as_grid(domain, f)
    tg = as_grid(domain, g) if g is not None else None
    res = _lib.out_double()
    _lib.call("blr_sq_dist", domain.ctx().bind(), ptr(tf), ptr(tg) if tg is not None else None,
              tf.numel(), C.byref(res))
    return domain.cell_volume * float(res.value)


def max_abs(domain: Domain, coeffs) -> float:
    """Max-norm of the spatial realization (full-grid include + reduction)."""
    g = include(domain, coeffs, check=False)
    return grid_max_abs(domain, g)


def grid_max_abs(domain: Domain, f) -> float:
    tf = as_grid(domain, f)
    res = _lib.out_double()
    _lib.call("blr_max_abs", domain.ctx().bind(), ptr(tf), tf.numel(), C.byref(res))
    return float(res.value)


def all_finite(domain: Domain, f) -> bool:
    tf = as_grid(domain, f)
    res = C.c_int(0)
    _lib.call("blr_all_finite", domain.ctx().bind(), ptr(tf), tf.numel(), C.byref(res))
    return bool(res.value)


def _domain_of(x) -> Domain:
    """A reduction-only context matching ``x``'s precision and device."""
    if isinstance(x, torch.Tensor) and x.is_cuda:
        dtype = "float32" if x.dtype in (torch.complex64, torch.float32) else "float64"
        return Domain((4,), (1,), dtype=dtype, device=x.device.index or 0)
    return Domain((4,), (1,))
