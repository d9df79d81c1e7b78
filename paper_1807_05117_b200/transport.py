"""Time integration of the band-limited transport equations on the B200.

Mirrors ``blreg/transport.py``: ``TimeFlow`` (device-resident node values),
quadrature, CFL control, and the RK4 integrators.  Each integrator is ONE
call into the sm_100a library, which runs the whole sweep (all RK4 stages,
pad-grid realizations, products and projections) on the caller's stream.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, spectral
from .domain import Domain
from .spectral import as_band, ptr


class CFLViolation(RuntimeError):
    """Raised when the transport CFL bound fails and refinement is disabled."""


# ---------------------------------------------------------------------------
# velocity flows (transport.py:36-126)
# ---------------------------------------------------------------------------

@dataclass(eq=False)
class TimeFlow:
    """Velocity flow on the nodes of [0, 1].

    ``values`` has shape ``(n_stored, d, *block)`` (``n_stored`` = 1 when
    stationary, else ``n_steps + 1``) and lives on the domain's device.
    """

    domain: Domain
    values: torch.Tensor
    n_steps: int
    stationary: bool

    def __post_init__(self):
        if self.n_steps < 1:
            raise ValueError("n_steps must be >= 1")
        self.values = as_band(self.domain, self.values)
        expected = 1 if self.stationary else self.n_steps + 1
        block = (self.domain.ndim,) + self.domain.block_shape
        if tuple(self.values.shape) != (expected,) + block:
            raise ValueError(
                f"flow values have shape {tuple(self.values.shape)}, expected {(expected,) + block}")

    @classmethod
    def zero(cls, domain: Domain, n_steps: int = 10, stationary: bool = True) -> "TimeFlow":
        n = 1 if stationary else n_steps + 1
        vals = torch.zeros((n, domain.ndim) + domain.block_shape, dtype=domain.cdtype,
                           device=domain.torch_device)
        return cls(domain, vals, n_steps, stationary)

    @property
    def n_nodes(self) -> int:
        return self.n_steps + 1

    @property
    def n_stored(self) -> int:
        return self.values.shape[0]

    def node(self, i: int) -> torch.Tensor:
        return self.values[0] if self.stationary else self.values[i]

    def sample(self, t: float) -> torch.Tensor:
        """Velocity at time t, linear between nodes (transport.py:77-86)."""
        if self.stationary:
            return self.values[0]
        s = min(max(t, 0.0), 1.0) * self.n_steps
        i = min(int(np.floor(s)), self.n_steps - 1)
        w = s - i
        if w == 0.0:
            return self.values[i]
        out = self.values[i].clone()
        _lib.call("blr_axpby", self.domain.ctx().bind(), w, ptr(self.values[i + 1]), 1.0 - w,
                  ptr(out), out.numel())
        return out

    def copy(self) -> "TimeFlow":
        return TimeFlow(self.domain, self.values.clone(), self.n_steps, self.stationary)

    def _like(self, values) -> "TimeFlow":
        return TimeFlow(self.domain, values, self.n_steps, self.stationary)

    def _check_compatible(self, other: "TimeFlow"):
        if (self.domain != other.domain or self.n_steps != other.n_steps
                or self.stationary != other.stationary):
            raise ValueError("incompatible flows")

    def lincomb(self, a: float, other: "TimeFlow | None" = None, b: float = 0.0) -> "TimeFlow":
        """``a * self + b * other`` in one kernel pass."""
        out = self.values.clone()
        h = self.domain.ctx().bind()
        if other is None:
            _lib.call("blr_axpby", h, 0.0, ptr(out), float(a), ptr(out), out.numel())
        else:
            self._check_compatible(other)
            _lib.call("blr_axpby", h, float(b), ptr(other.values), float(a), ptr(out), out.numel())
        return self._like(out)

    def __add__(self, other: "TimeFlow") -> "TimeFlow":
        return self.lincomb(1.0, other, 1.0)

    def __sub__(self, other: "TimeFlow") -> "TimeFlow":
        return self.lincomb(1.0, other, -1.0)

    def __mul__(self, scalar: float) -> "TimeFlow":
        return self.lincomb(float(scalar))

    __rmul__ = __mul__

    def map_nodes(self, fn) -> "TimeFlow":
        out = torch.empty_like(self.values)
        for i in range(self.n_stored):
            out[i] = fn(self.values[i])
        return self._like(out)

    def max_speed(self) -> float:
        """max over nodes of max|iota(v_i)| on the image grid."""
        return spectral.max_abs(self.domain, self.values)

    def max_divergence(self) -> float:
        dom = self.domain
        div = torch.empty((self.n_stored,) + dom.block_shape, dtype=dom.cdtype, device=dom.torch_device)
        _lib.call("blr_divergence", dom.ctx().bind(), ptr(self.values), self.n_stored, ptr(div))
        return float(div.abs().max())

    def numpy(self) -> np.ndarray:
        return self.values.detach().cpu().numpy()


def time_weights(n_steps: int, rule: str = "trapezoid") -> np.ndarray:
    """Quadrature weights on the n_steps + 1 nodes (transport.py:129-144)."""
    dt = 1.0 / n_steps
    if rule == "trapezoid":
        w = np.full(n_steps + 1, dt)
        w[0] = w[-1] = dt / 2.0
        return w
    if rule == "simpson":
        if n_steps % 2 != 0:
            raise ValueError("simpson weights need an even number of steps")
        w = np.empty(n_steps + 1)
        w[0::2] = 2.0
        w[1::2] = 4.0
        w[0] = w[-1] = 1.0
        return w * (dt / 3.0)
    raise ValueError(f"unknown quadrature rule {rule!r}")


def flow_inner(a: TimeFlow, b: TimeFlow, rule: str = "trapezoid") -> float:
    """Time-weighted inner product (transport.py:147-153), one device reduction per node."""
    a._check_compatible(b)
    dom = a.domain
    h = dom.ctx().bind()
    res = _lib.out_double()
    if a.stationary:
        _lib.call("blr_inner", h, ptr(a.values), ptr(b.values), a.values.numel(), C.byref(res))
        return float(res.value)
    w, keep = _lib.double_array(time_weights(a.n_steps, rule))
    n = a.values[0].numel()
    _lib.call("blr_inner_nodes", h, ptr(a.values), ptr(b.values), a.n_nodes, n, w, C.byref(res))
    del keep
    return float(res.value)


def flow_max_abs(flow: TimeFlow) -> float:
    return flow.max_speed()


# ---------------------------------------------------------------------------
# CFL monitoring (transport.py:165-199)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class CFLReport:
    number: float
    limit: float
    passed: bool
    suggested_steps: int


def check_cfl(flow: TimeFlow, n_steps: int | None = None, limit: float = 0.5) -> CFLReport:
    if n_steps is None:
        n_steps = flow.n_steps
    h_min = min(flow.domain.spacing)
    speed = flow.max_speed()
    number = speed / (n_steps * h_min)
    if speed == 0.0:
        return CFLReport(0.0, limit, True, n_steps)
    suggested = max(1, int(np.ceil(speed / (limit * h_min))))
    return CFLReport(number, limit, number <= limit, max(suggested, 1))


def resolve_substeps(flow: TimeFlow, limit: float, auto_refine: bool) -> int:
    report = check_cfl(flow, limit=limit)
    if report.passed:
        return 1
    if not auto_refine:
        raise CFLViolation(
            f"CFL number {report.number:.3g} exceeds {limit}; "
            f"needs at least {report.suggested_steps} time steps")
    return int(np.ceil(report.suggested_steps / flow.n_steps))


# ---------------------------------------------------------------------------
# integrators (transport.py:351-465)
# ---------------------------------------------------------------------------

def _nodes(dom: Domain, n_nodes: int, comps: int | None) -> torch.Tensor:
    lead = (n_nodes,) if comps is None else (n_nodes, comps)
    return torch.empty(lead + dom.block_shape, dtype=dom.cdtype, device=dom.torch_device)


def du_cache_shape(v: TimeFlow, substeps: int) -> tuple:
    dom = v.domain
    return (4 * v.n_steps * substeps, dom.ndim * dom.ndim) + dom.pad


def du_cache_bytes(v: TimeFlow, substeps: int) -> int:
    el = 8 if v.domain.dtype == "float64" else 4
    return int(np.prod(du_cache_shape(v, substeps))) * el


def integrate_forward_map(v: TimeFlow, substeps: int = 1, du_cache: torch.Tensor | None = None):
    """Displacement nodes of phi~ = id + u (transport.py:351-363).

    ``du_cache`` (optional, ``du_cache_shape``): filled with the pad-grid
    realizations of D(u) at every RK4 stage for ``integrate_state_tangents``.
    """
    dom = v.domain
    out = _nodes(dom, v.n_nodes, dom.ndim)
    _lib.call("blr_forward_map", dom.ctx().bind(), ptr(v.values), v.n_stored, v.n_steps,
              int(substeps), ptr(out), ptr(du_cache) if du_cache is not None else None)
    return out


def integrate_inverse_map_and_volume(v: TimeFlow, substeps: int = 1):
    """psi~ and J~ nodes, integrated backward from the identity (transport.py:366-383)."""
    dom = v.domain
    psi = _nodes(dom, v.n_nodes, dom.ndim)
    vol = _nodes(dom, v.n_nodes, None)
    _lib.call("blr_inverse_map_and_volume", dom.ctx().bind(), ptr(v.values), v.n_stored,
              v.n_steps, int(substeps), ptr(psi), ptr(vol))
    return psi, vol


def integrate_state_tangents(v: TimeFlow, dv: TimeFlow, substeps: int = 1, with_volume: bool = True,
                             with_inverse: bool = True, with_forward: bool = True,
                             du_cache: torch.Tensor | None = None, final_only: bool = False):
    """(dphi, dpsi, dvol) tangent node arrays (transport.py:386-432).

    ``final_only`` records just the last forward-tangent node (dphi has one
    node): the Gauss-Newton deformation HVP reads only dphi[-1]."""
    v._check_compatible(dv)
    dom = v.domain
    dphi = _nodes(dom, 1 if final_only else v.n_nodes, dom.ndim) if with_forward else None
    dpsi = _nodes(dom, v.n_nodes, dom.ndim) if with_inverse else None
    dvol = _nodes(dom, v.n_nodes, None) if (with_inverse and with_volume) else None
    flags = (1 if with_forward else 0) | (2 if with_inverse else 0) | (4 if dvol is not None else 0)
    if final_only and with_forward:
        flags |= 8
    _lib.call("blr_state_tangents", dom.ctx().bind(), ptr(v.values), ptr(dv.values), v.n_stored,
              v.n_steps, int(substeps), flags, ptr(du_cache) if du_cache is not None else None,
              ptr(dphi) if dphi is not None else None, ptr(dpsi) if dpsi is not None else None,
              ptr(dvol) if dvol is not None else None)
    return dphi, dpsi, dvol


def integrate_momentum(v: TimeFlow, momentum_end, substeps: int = 1):
    """Backward conservative transport of a vector momentum (transport.py:435-445)."""
    dom = v.domain
    rho_end = as_band(dom, momentum_end)
    out = _nodes(dom, v.n_nodes, dom.ndim)
    _lib.call("blr_momentum", dom.ctx().bind(), ptr(v.values), v.n_stored, v.n_steps,
              int(substeps), ptr(rho_end), ptr(out))
    return out


def integrate_momentum_tangent(v: TimeFlow, dv: TimeFlow, momentum_end, tangent_end,
                               substeps: int = 1, gauss_newton: bool = False, want_base: bool = True):
    """Momentum and its tangent (transport.py:448-465)."""
    v._check_compatible(dv)
    dom = v.domain
    rho_end, drho_end = as_band(dom, momentum_end), as_band(dom, tangent_end)
    rho = _nodes(dom, v.n_nodes, dom.ndim) if (want_base or not gauss_newton) else None
    drho = _nodes(dom, v.n_nodes, dom.ndim)
    _lib.call("blr_momentum_tangent", dom.ctx().bind(), ptr(v.values), ptr(dv.values), v.n_stored,
              v.n_steps, int(substeps), ptr(rho_end), ptr(drho_end), int(bool(gauss_newton)),
              ptr(rho) if rho is not None else None, ptr(drho))
    return rho, drho


# ---------------------------------------------------------------------------
# trajectory cache (transport.py:472-494)
# ---------------------------------------------------------------------------

@dataclass(eq=False)
class TrajectoryCache:
    """Node trajectories retained for gradient and Hessian-vector reuse."""

    velocity: TimeFlow
    substeps: int
    forward: torch.Tensor
    inverse: torch.Tensor | None = None
    volume: torch.Tensor | None = None
    momentum: torch.Tensor | None = None
    momentum_end: torch.Tensor | None = None

    def assert_matches(self, v: TimeFlow):
        if v is self.velocity:
            return
        if (v.domain != self.velocity.domain or v.n_steps != self.velocity.n_steps
                or v.stationary != self.velocity.stationary
                or not torch.equal(v.values, self.velocity.values)):
            raise ValueError("trajectory cache does not match this velocity flow")
