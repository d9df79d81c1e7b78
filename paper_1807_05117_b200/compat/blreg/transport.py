"""Flows and transport (reference ``transport.py``) with host (numpy) flows.

``TimeFlow`` keeps the reference's numpy container semantics
(``transport.py:36-126``); every integrator and the inner products run on
the device (``paper_1807_05117_b200.transport``) and return numpy.
"""

from dataclasses import dataclass

import numpy as np

from paper_1807_05117_b200 import transport as _t
from paper_1807_05117_b200.transport import CFLReport, CFLViolation, time_weights  # noqa: F401

from . import spectral
from ._conv import dev, host


@dataclass
class TimeFlow:
    domain: object
    values: np.ndarray
    n_steps: int
    stationary: bool

    def __post_init__(self):
        if self.n_steps < 1:
            raise ValueError("n_steps must be >= 1")
        self.values = np.asarray(self.values)
        expected = 1 if self.stationary else self.n_steps + 1
        block = (self.domain.ndim,) + self.domain.block_shape
        if self.values.shape != (expected,) + block:
            raise ValueError(f"flow values have shape {self.values.shape}, expected {(expected,) + block}")

    # -- host <-> device -------------------------------------------------------
    def device(self) -> "_t.TimeFlow":
        return _t.TimeFlow(self.domain, dev(self.domain, self.values, True), self.n_steps, self.stationary)

    @classmethod
    def from_device(cls, flow: "_t.TimeFlow") -> "TimeFlow":
        return cls(flow.domain, host(flow.values), flow.n_steps, flow.stationary)

    # -- reference container API -------------------------------------------------
    @classmethod
    def zero(cls, domain, n_steps: int = 10, stationary: bool = True) -> "TimeFlow":
        n = 1 if stationary else n_steps + 1
        return cls(domain, np.zeros((n, domain.ndim) + domain.block_shape, dtype=np.complex128), n_steps,
                   stationary)

    @property
    def n_nodes(self) -> int:
        return self.n_steps + 1

    @property
    def n_stored(self) -> int:
        return self.values.shape[0]

    def node(self, i: int) -> np.ndarray:
        return self.values[0] if self.stationary else self.values[i]

    def sample(self, t: float) -> np.ndarray:
        return host(self.device().sample(t))

    def copy(self) -> "TimeFlow":
        return TimeFlow(self.domain, self.values.copy(), self.n_steps, self.stationary)

    def _like(self, values) -> "TimeFlow":
        return TimeFlow(self.domain, values, self.n_steps, self.stationary)

    def _check_compatible(self, other: "TimeFlow"):
        if (self.domain != other.domain or self.n_steps != other.n_steps
                or self.stationary != other.stationary):
            raise ValueError("incompatible flows")

    def __add__(self, other: "TimeFlow") -> "TimeFlow":
        self._check_compatible(other)
        return self._like(self.values + other.values)

    def __sub__(self, other: "TimeFlow") -> "TimeFlow":
        self._check_compatible(other)
        return self._like(self.values - other.values)

    def __mul__(self, scalar: float) -> "TimeFlow":
        return self._like(self.values * scalar)

    __rmul__ = __mul__

    def map_nodes(self, fn) -> "TimeFlow":
        out = np.empty_like(self.values)
        for i in range(self.n_stored):
            out[i] = fn(self.values[i])
        return self._like(out)

    def max_speed(self) -> float:
        return self.device().max_speed()

    def max_divergence(self) -> float:
        return self.device().max_divergence()


def _d(flow):
    return flow.device() if isinstance(flow, TimeFlow) else flow


def flow_inner(a, b, rule: str = "trapezoid") -> float:
    return _t.flow_inner(_d(a), _d(b), rule)


def flow_max_abs(flow) -> float:
    return _t.flow_max_abs(_d(flow))


def check_cfl(flow, n_steps=None, limit: float = 0.5) -> CFLReport:
    return _t.check_cfl(_d(flow), n_steps, limit)


def resolve_substeps(flow, limit: float, auto_refine: bool) -> int:
    return _t.resolve_substeps(_d(flow), limit, auto_refine)


def integrate_forward_map(v, substeps: int = 1):
    return host(_t.integrate_forward_map(_d(v), substeps))


def integrate_inverse_map_and_volume(v, substeps: int = 1):
    return host(_t.integrate_inverse_map_and_volume(_d(v), substeps))


def integrate_state_tangents(v, dv, substeps: int = 1, with_volume: bool = True, with_inverse: bool = True):
    out = _t.integrate_state_tangents(_d(v), _d(dv), substeps, with_volume=with_volume,
                                      with_inverse=with_inverse)
    return tuple(host(x) if x is not None else None for x in out)


def integrate_momentum(v, momentum_end, substeps: int = 1):
    dv = _d(v)
    return host(_t.integrate_momentum(dv, dev(dv.domain, momentum_end, True), substeps))


def integrate_momentum_tangent(v, dv, momentum_end, tangent_end, substeps: int = 1, gauss_newton: bool = False):
    vd = _d(v)
    out = _t.integrate_momentum_tangent(vd, _d(dv), dev(vd.domain, momentum_end, True),
                                        dev(vd.domain, tangent_end, True), substeps, gauss_newton=gauss_newton)
    return tuple(host(x) if x is not None else None for x in out)


class TrajectoryCache:
    """Host view of a device trajectory cache: arrays copied on first access."""

    def __init__(self, cache, velocity: TimeFlow):
        self._c = cache
        self.velocity = velocity
        self.substeps = cache.substeps
        self._h = {}

    def _get(self, name):
        if name not in self._h:
            val = getattr(self._c, name)
            self._h[name] = host(val) if val is not None else None
        return self._h[name]

    forward = property(lambda self: self._get("forward"))
    inverse = property(lambda self: self._get("inverse"))
    volume = property(lambda self: self._get("volume"))
    momentum = property(lambda self: self._get("momentum"))
    momentum_end = property(lambda self: self._get("momentum_end"))

    def assert_matches(self, v):
        if v is self.velocity:
            return
        if (v.domain != self.velocity.domain or v.n_steps != self.velocity.n_steps
                or v.stationary != self.velocity.stationary
                or not np.array_equal(v.values, self.velocity.values)):
            raise ValueError("trajectory cache does not match this velocity flow")
