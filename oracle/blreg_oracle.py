"""CPU ORACLE — test infrastructure only, never the product.

This module is a numpy/scipy restatement of the reference package ``blreg``
(``/root/reference/pkg/src/blreg``) for the Gauss-Newton-Krylov hot path:
band-limited spectral algebra, RK4 spectral transport with tangents, periodic
warps and stencils, the two registration objectives (energy, gradient, GN and
Newton Hessian-vector products) and the PCG / Armijo solver.  Every function
cites the reference ``file:line`` it restates.

Who may use it: ``tests/``, ``__graft_entry__.smoke()`` (as the checker) and
``bench.py`` (the ``cpu_baseline`` leg and ``--impl reference``).  The product
package ``paper_1807_05117_b200`` never imports it.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference in the
build container and stores inputs/outputs as ``.npz`` fixtures;
``tests/test_oracle_golden.py`` checks this oracle against every fixture.

Formulation differences from the reference (same mathematics, rounding-level
differences only): band blocks are realized with real-to-complex transforms
(``irfftn``/``rfftn``) on the Hermitian half spectrum instead of complex
``ifftn(...).real``; the pad grid defaults to the reference's
``next_fast_len(4K+1)`` but any ``P >= 3K+1`` can be requested (exact, since
every product on the pad grid is bilinear in K-band fields).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace
from functools import lru_cache

import numpy as np
import scipy.fft
from scipy import ndimage

TWO_PI = 2.0 * np.pi
WORKERS = 1  # scipy.fft worker threads; bench.py raises it for the threaded baseline


# ---------------------------------------------------------------------------
# domain (domain.py:19-97)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Dom:
    """Restates ``Domain`` (domain.py:19-63) without the field helpers."""
    shape: tuple
    bandwidth: tuple
    alpha: float = 0.02
    order: int = 2
    symbol: str = "discrete"
    pad: tuple | None = None  # None -> reference pad next_fast_len(4K+1)

    def __post_init__(self):
        object.__setattr__(self, "shape", tuple(int(n) for n in self.shape))
        object.__setattr__(self, "bandwidth", tuple(int(k) for k in self.bandwidth))
        if len(self.shape) not in (1, 2, 3) or len(self.bandwidth) != len(self.shape):
            raise ValueError("bad domain")
        for n, k in zip(self.shape, self.bandwidth):
            if n < 2 or not 1 <= k <= n // 2:
                raise ValueError("bad bandwidth")
        if not self.alpha > 0 or int(self.order) < 1:
            raise ValueError("bad metric")
        if self.symbol not in ("discrete", "continuous"):
            raise ValueError("bad symbol")
        if self.pad is not None:
            object.__setattr__(self, "pad", tuple(int(p) for p in self.pad))
            for p, k in zip(self.pad, self.bandwidth):
                if p < 3 * k + 1:
                    raise ValueError("pad grid must have at least 3K+1 points")

    @property
    def ndim(self):
        return len(self.shape)

    @property
    def block(self):  # domain.py:73-76
        return tuple(2 * k + 1 for k in self.bandwidth)

    @property
    def h(self):  # domain.py:69-71
        return tuple(1.0 / n for n in self.shape)

    @property
    def cell(self):  # domain.py:78-80
        return float(np.prod(self.h))

    @property
    def pad_shape(self):  # spectral.py:142-145
        if self.pad is not None:
            return self.pad
        return tuple(scipy.fft.next_fast_len(2 * (b - 1) + 1) for b in self.block)

    def zeros_vec(self, lead=()):
        return np.zeros(tuple(lead) + (self.ndim,) + self.block, dtype=np.complex128)


def freqs_of(m: int) -> np.ndarray:
    """Wrap-order integer frequencies of a block axis (domain.py:93-97)."""
    k = (m - 1) // 2
    return np.concatenate([np.arange(0, k + 1), np.arange(-k, 0)]).astype(np.int64)


def _bcast(vec, ax, d):
    sh = [1] * d
    sh[ax] = vec.size
    return vec.reshape(sh)


# ---------------------------------------------------------------------------
# symmetry (spectral.py:37-56)
# ---------------------------------------------------------------------------

def conj_reverse(c: np.ndarray, d: int) -> np.ndarray:
    """conj(c(-k)) on the trailing d axes (spectral.py:37-42)."""
    out = c
    for ax in range(c.ndim - d, c.ndim):
        m = c.shape[ax]
        out = np.take(out, (-np.arange(m)) % m, axis=ax)
    return np.conj(out)


def symmetrize(c: np.ndarray, d: int) -> np.ndarray:
    """Hermitian part (spectral.py:45-47)."""
    return 0.5 * (c + conj_reverse(c, d))


def symmetry_error(c: np.ndarray, d: int) -> float:
    """spectral.py:50-56."""
    scale = float(np.max(np.abs(c))) if c.size else 0.0
    if scale == 0.0:
        return 0.0
    return float(np.max(np.abs(c - conj_reverse(c, d)))) / scale


# ---------------------------------------------------------------------------
# include / project via the Hermitian half spectrum (spectral.py:63-135)
# ---------------------------------------------------------------------------

@lru_cache(maxsize=None)
def _embed(block: tuple, grid: tuple):
    """Bin map + gather weights (spectral.py:63-86)."""
    bins, wts, coll = [], [], False
    for m, p in zip(block, grid):
        b = np.mod(freqs_of(m), p)
        cnt = np.bincount(b, minlength=p)
        coll = coll or bool(np.any(cnt > 1))
        bins.append(b)
        wts.append(1.0 / cnt[b])
    w = wts[0]
    for e in wts[1:]:
        w = np.multiply.outer(w, e)
    return tuple(bins), w, coll


def include(dom: Dom, c: np.ndarray, grid=None, check=True) -> np.ndarray:
    """Band block(s) -> real grid field(s) (spectral.py:89-119).

    Zero-pad into the half spectrum of the grid and apply an unnormalized
    real inverse DFT (equal to ``ifftn(...).real * prod(grid)`` for Hermitian
    blocks).
    """
    grid = tuple(dom.shape if grid is None else grid)
    d = dom.ndim
    if c.shape[-d:] != dom.block:
        raise ValueError("block shape mismatch")
    if check and symmetry_error(c, d) > 1e-10:
        raise ValueError("coefficients violate conjugate symmetry; spectrum is corrupted")
    lead = c.shape[:-d]
    comps = c.reshape((-1,) + dom.block)
    bins, _, coll = _embed(dom.block, grid)
    half = grid[-1] // 2 + 1
    keep = bins[-1] < half
    zb = bins[-1][keep]
    H = np.zeros((comps.shape[0],) + grid[:-1] + (half,), dtype=np.complex128)
    src = comps[..., keep]
    ix = np.ix_(*bins[:-1], zb)
    if coll:
        for i in range(comps.shape[0]):
            np.add.at(H[i], ix, src[i])
    else:
        H[(slice(None),) + ix] = src
    axes = tuple(range(1, d + 1))
    out = scipy.fft.irfftn(H, s=grid, axes=axes, norm="forward", workers=WORKERS)
    return np.ascontiguousarray(out.reshape(lead + grid))


def project(dom: Dom, f: np.ndarray, grid=None) -> np.ndarray:
    """Real grid field(s) -> band block(s): forward DFT/prod, gather, symmetrize
    (spectral.py:122-135)."""
    grid = tuple(dom.shape if grid is None else grid)
    d = dom.ndim
    lead = f.shape[:-d]
    comps = f.reshape((-1,) + grid)
    axes = tuple(range(1, d + 1))
    H = scipy.fft.rfftn(comps, axes=axes, norm="forward", workers=WORKERS)
    bins, w, _ = _embed(dom.block, grid)
    half = grid[-1] // 2 + 1
    # value at bin b of the full spectrum: H[b] if b_z < half else conj(H[-b])
    g = np.empty((comps.shape[0],) + dom.block, dtype=np.complex128)
    fz = freqs_of(dom.block[-1])
    bz = bins[-1]
    lo = bz < half
    g[..., lo] = H[(slice(None),) + np.ix_(*bins[:-1], bz[lo])]
    if np.any(~lo):
        mb = [(-b) % p for b, p in zip(bins[:-1], grid[:-1])]
        mz = (-bz[~lo]) % grid[-1]
        g[..., ~lo] = np.conj(H[(slice(None),) + np.ix_(*mb, mz)])
    del fz
    out = symmetrize(g * w, d)
    return np.ascontiguousarray(out.reshape(lead + dom.block))


def to_pad(dom, c):  # spectral.py:148-149
    return include(dom, c, dom.pad_shape, check=False)


def from_pad(dom, f):  # spectral.py:152-153
    return project(dom, f, dom.pad_shape)


# ---------------------------------------------------------------------------
# diagonal operators (spectral.py:242-328, 339-425)
# ---------------------------------------------------------------------------

def kvecs(dom):
    d = dom.ndim
    return [_bcast(TWO_PI * freqs_of(m).astype(np.float64), ax, d) for ax, m in enumerate(dom.block)]


def base_symbol(dom):
    """1 + alpha * sum_j s_j(k) (spectral.py:242-257)."""
    acc = np.zeros(dom.block)
    for ax, (m, n) in enumerate(zip(dom.block, dom.shape)):
        f = freqs_of(m)
        if dom.symbol == "discrete":
            t = 2.0 * n * n * (1.0 - np.cos(TWO_PI * f / n))
        else:
            t = (TWO_PI * f) ** 2
        acc = acc + _bcast(t, ax, dom.ndim)
    return 1.0 + dom.alpha * acc


def helmholtz(dom, c):  # spectral.py:265-267
    return c * (base_symbol(dom) ** dom.order)


def inv_helmholtz(dom, c):  # spectral.py:270-272
    return c * (base_symbol(dom) ** (-dom.order))


def grad(dom, s):  # spectral.py:275-281
    return np.stack([1j * k * s for k in kvecs(dom)])


def div(dom, v):  # spectral.py:284-289
    out = np.zeros(dom.block, dtype=np.complex128)
    for ax, k in enumerate(kvecs(dom)):
        out += 1j * k * v[ax]
    return out


def jac(dom, v):  # spectral.py:292-300 ; out[i, j] = d_j v_i
    ks = kvecs(dom)
    return np.stack([np.stack([1j * ks[j] * v[i] for j in range(dom.ndim)]) for i in range(dom.ndim)])


def leray(dom, v):  # spectral.py:312-328
    dv = div(dom, v)
    lap = np.zeros(dom.block)
    for k in kvecs(dom):
        lap = lap - k ** 2
    p = np.zeros_like(dv)
    nz = lap != 0.0
    p[nz] = dv[nz] / lap[nz]
    return v - grad(dom, p)


def inner(a, b):  # spectral.py:335-337
    return float(np.real(np.vdot(b, a)))


def grid_norm2(dom, f):  # spectral.py:344-345
    return dom.cell * float(np.sum(f * f))


def max_abs(dom, c):  # spectral.py:348-350
    return float(np.max(np.abs(include(dom, c, check=False))))


def conv_matvec(dom, M, v, transpose=False):  # spectral.py:194-200
    d = dom.ndim
    mg = to_pad(dom, M.reshape((d * d,) + dom.block)).reshape((d, d) + dom.pad_shape)
    vg = to_pad(dom, v)
    spec = "ji...,j...->i..." if transpose else "ij...,j...->i..."
    return from_pad(dom, np.einsum(spec, mg, vg))


def conv_scalar(dom, a, b):  # spectral.py:181-184
    return from_pad(dom, to_pad(dom, a) * to_pad(dom, b))


# ---------------------------------------------------------------------------
# flows (transport.py:36-158)
# ---------------------------------------------------------------------------

@dataclass
class Flow:
    """Restates ``TimeFlow`` (transport.py:36-126)."""
    dom: Dom
    values: np.ndarray
    n_steps: int
    stationary: bool

    def sample(self, t):  # transport.py:77-86
        if self.stationary:
            return self.values[0]
        s = min(max(t, 0.0), 1.0) * self.n_steps
        i = min(int(np.floor(s)), self.n_steps - 1)
        w = s - i
        if w == 0.0:
            return self.values[i]
        return (1.0 - w) * self.values[i] + w * self.values[i + 1]

    @property
    def n_nodes(self):
        return self.n_steps + 1

    def like(self, values):
        return Flow(self.dom, values, self.n_steps, self.stationary)

    def map_nodes(self, fn):
        return self.like(np.stack([fn(x) for x in self.values]))

    def max_speed(self):  # transport.py:119-120
        return max(max_abs(self.dom, x) for x in self.values)

    def max_divergence(self):  # transport.py:122-126
        return max(float(np.max(np.abs(div(self.dom, x)))) for x in self.values)


def time_weights(n, rule="trapezoid"):  # transport.py:129-144
    dt = 1.0 / n
    if rule == "trapezoid":
        w = np.full(n + 1, dt)
        w[0] = w[-1] = dt / 2.0
        return w
    if rule == "simpson":
        if n % 2:
            raise ValueError("simpson weights need an even number of steps")
        w = np.empty(n + 1)
        w[0::2], w[1::2] = 2.0, 4.0
        w[0] = w[-1] = 1.0
        return w * (dt / 3.0)
    raise ValueError(rule)


def flow_inner(a: Flow, b: Flow, rule="trapezoid"):  # transport.py:147-153
    if a.stationary:
        return inner(a.values[0], b.values[0])
    w = time_weights(a.n_steps, rule)
    return float(sum(w[i] * inner(a.values[i], b.values[i]) for i in range(a.n_nodes)))


class CFLViolation(RuntimeError):
    pass


def cfl(flow: Flow, limit=0.5):
    """(number, passed, suggested) (transport.py:173-186)."""
    hmin = min(flow.dom.h)
    speed = flow.max_speed()
    number = speed / (flow.n_steps * hmin)
    if speed == 0.0:
        return 0.0, True, flow.n_steps
    sug = max(1, int(np.ceil(speed / (limit * hmin))))
    return number, number <= limit, sug


def substeps_for(flow: Flow, limit=0.5, auto_refine=True):  # transport.py:189-199
    number, ok, sug = cfl(flow, limit)
    if ok:
        return 1
    if not auto_refine:
        raise CFLViolation(f"CFL number {number:.3g} exceeds {limit}")
    return int(np.ceil(sug / flow.n_steps))


# ---------------------------------------------------------------------------
# right-hand sides (transport.py:206-303)
# ---------------------------------------------------------------------------

def _mv(M, v):
    return np.einsum("ij...,j...->i...", M, v)


def rhs_map(dom, u, vt):  # transport.py:206-213 : -(v + Du * v)
    d = dom.ndim
    g = to_pad(dom, np.concatenate([jac(dom, u).reshape((d * d,) + dom.block), vt]))
    J = g[:d * d].reshape((d, d) + g.shape[1:])
    return -(vt + from_pad(dom, _mv(J, g[d * d:])))


def rhs_map_tangent(dom, u, du, vt, dvt):  # transport.py:216-228
    d = dom.ndim
    st = np.concatenate([jac(dom, u).reshape((d * d,) + dom.block),
                         jac(dom, du).reshape((d * d,) + dom.block), vt, dvt])
    g = to_pad(dom, st)
    sh = (d, d) + g.shape[1:]
    J, dJ = g[:d * d].reshape(sh), g[d * d:2 * d * d].reshape(sh)
    V, dV = g[2 * d * d:2 * d * d + d], g[2 * d * d + d:]
    return -(dvt + from_pad(dom, _mv(dJ, V) + _mv(J, dV)))


def rhs_volume(dom, J, vt):  # transport.py:231-241
    d = dom.ndim
    g = to_pad(dom, np.concatenate([vt, grad(dom, J), J[None], div(dom, vt)[None]]))
    return from_pad(dom, -np.einsum("a...,a...->...", g[:d], g[d:2 * d]) - g[2 * d] * g[2 * d + 1])


def rhs_volume_tangent(dom, J, dJ, vt, dvt):  # transport.py:244-261
    d = dom.ndim
    st = np.concatenate([vt, dvt, grad(dom, J), grad(dom, dJ), J[None], dJ[None],
                         div(dom, vt)[None], div(dom, dvt)[None]])
    g = to_pad(dom, st)
    V, dV, G, dG = g[:d], g[d:2 * d], g[2 * d:3 * d], g[3 * d:4 * d]
    r = (-np.einsum("a...,a...->...", dV, G) - np.einsum("a...,a...->...", V, dG)
         - g[4 * d + 1] * g[4 * d + 2] - g[4 * d] * g[4 * d + 3])
    return from_pad(dom, r)


def _flux_div(dom, fl):
    """-(row divergence) of projected flux blocks (transport.py:264-274)."""
    d = dom.ndim
    ks = kvecs(dom)
    out = np.zeros(fl.shape[:-d - 2] + (d,) + dom.block, dtype=np.complex128)
    blk = (slice(None),) * d
    for i in range(d):
        for j in range(d):
            out[(Ellipsis, i) + blk] += 1j * ks[j] * fl[(Ellipsis, i, j) + blk]
    return out


def _fl(dom, F):
    d = dom.ndim
    lead = F.shape[:-d]
    return from_pad(dom, F.reshape((-1,) + dom.pad_shape)).reshape(lead + dom.block)


def rhs_momentum(dom, rho, vt):  # transport.py:277-281
    d = dom.ndim
    g = to_pad(dom, np.concatenate([rho, vt]))
    F = np.einsum("i...,j...->ij...", g[:d], g[d:])
    return -_flux_div(dom, _fl(dom, F))


def rhs_momentum_pair(dom, rho, drho, vt, dvt):  # transport.py:284-303
    d = dom.ndim
    parts = [rho, drho, vt] + ([dvt] if dvt is not None else [])
    g = to_pad(dom, np.concatenate(parts))
    R, dR, V = g[:d], g[d:2 * d], g[2 * d:3 * d]
    base = np.einsum("i...,j...->ij...", R, V)
    tan = np.einsum("i...,j...->ij...", dR, V)
    if dvt is not None:
        tan = tan + np.einsum("i...,j...->ij...", R, g[3 * d:])
    out = _flux_div(dom, _fl(dom, np.stack([base, tan])))
    return -out[0], -out[1]


# ---------------------------------------------------------------------------
# RK4 driver and integrators (transport.py:310-465)
# ---------------------------------------------------------------------------

def rk4(flow: Flow, state0, rhs, forward, substeps):
    """Classical RK4 over all node intervals, nodes recorded ascending
    (transport.py:310-344)."""
    n = flow.n_steps
    h = ((1.0 if forward else -1.0) / n) / substeps
    nodes = range(n) if forward else range(n, 0, -1)
    st = tuple(np.copy(s) for s in state0)
    rec = [st]
    for node in nodes:
        t0 = node / n
        for k in range(substeps):
            t = t0 + k * h
            a, b, c = flow.sample(t), flow.sample(t + 0.5 * h), flow.sample(t + h)
            k1 = rhs(t, st, a)
            k2 = rhs(t + 0.5 * h, tuple(s + 0.5 * h * q for s, q in zip(st, k1)), b)
            k3 = rhs(t + 0.5 * h, tuple(s + 0.5 * h * q for s, q in zip(st, k2)), b)
            k4 = rhs(t + h, tuple(s + h * q for s, q in zip(st, k3)), c)
            st = tuple(s + (h / 6.0) * (q1 + 2.0 * q2 + 2.0 * q3 + q4)
                       for s, q1, q2, q3, q4 in zip(st, k1, k2, k3, k4))
        rec.append(tuple(np.copy(s) for s in st))
    if not forward:
        rec.reverse()
    return [np.stack([r[j] for r in rec]) for j in range(len(state0))]


def _unit_scalar(dom):
    one = np.zeros(dom.block, dtype=np.complex128)
    one[(0,) * dom.ndim] = 1.0
    return one


def forward_map(v: Flow, substeps=1):  # transport.py:351-363
    dom = v.dom
    return rk4(v, (dom.zeros_vec(),), lambda t, s, vt: (rhs_map(dom, s[0], vt),), True, substeps)[0]


def inverse_map_and_volume(v: Flow, substeps=1):  # transport.py:366-383
    dom = v.dom
    res = rk4(v, (dom.zeros_vec(), _unit_scalar(dom)),
              lambda t, s, vt: (rhs_map(dom, s[0], vt), rhs_volume(dom, s[1], vt)),
              False, substeps)
    return res[0], res[1]


def state_tangents(v: Flow, dv: Flow, substeps=1, with_volume=True, with_inverse=True):
    """transport.py:386-432."""
    dom = v.dom

    def fwd(t, s, vt):
        dvt = dv.sample(t)
        return rhs_map(dom, s[0], vt), rhs_map_tangent(dom, s[0], s[1], vt, dvt)

    dphi = rk4(v, (dom.zeros_vec(), dom.zeros_vec()), fwd, True, substeps)[1]
    if not with_inverse:
        return dphi, None, None
    if with_volume:
        def bwd(t, s, vt):
            dvt = dv.sample(t)
            w, dw, J, dJ = s
            return (rhs_map(dom, w, vt), rhs_map_tangent(dom, w, dw, vt, dvt),
                    rhs_volume(dom, J, vt), rhs_volume_tangent(dom, J, dJ, vt, dvt))
        res = rk4(v, (dom.zeros_vec(), dom.zeros_vec(), _unit_scalar(dom),
                      np.zeros(dom.block, complex)), bwd, False, substeps)
        return dphi, res[1], res[3]

    def bwd2(t, s, vt):
        dvt = dv.sample(t)
        return rhs_map(dom, s[0], vt), rhs_map_tangent(dom, s[0], s[1], vt, dvt)
    res = rk4(v, (dom.zeros_vec(), dom.zeros_vec()), bwd2, False, substeps)
    return dphi, res[1], None


def momentum(v: Flow, rho_end, substeps=1):  # transport.py:435-445
    dom = v.dom
    return rk4(v, (rho_end.copy(),), lambda t, s, vt: (rhs_momentum(dom, s[0], vt),),
               False, substeps)[0]


def momentum_tangent(v: Flow, dv: Flow, rho_end, drho_end, substeps=1, gauss_newton=False):
    """transport.py:448-465."""
    dom = v.dom

    def rhs(t, s, vt):
        dvt = None if gauss_newton else dv.sample(t)
        return rhs_momentum_pair(dom, s[0], s[1], vt, dvt)

    res = rk4(v, (rho_end.copy(), drho_end.copy()), rhs, False, substeps)
    return res[0], res[1]


# ---------------------------------------------------------------------------
# full-grid operations (gridops.py:21-131)
# ---------------------------------------------------------------------------

def sample_coords(dom, disp):  # gridops.py:21-29
    out = np.empty_like(disp)
    for ax, n in enumerate(dom.shape):
        out[ax] = _bcast(np.arange(n, dtype=np.float64), ax, dom.ndim) + disp[ax] * n
    return out


def warp(dom, f, disp, interp="linear"):
    """Periodic evaluation of f at x + u(x) (gridops.py:32-48); scipy's
    ``map_coordinates(mode="grid-wrap")`` is the reference's own evaluator."""
    if interp == "fourier":
        return fourier_warp(dom, f, disp)
    order = {"nearest": 0, "linear": 1, "cubic": 3}.get(interp)
    if order is None:
        raise ValueError(f"unknown interpolation {interp!r}")
    return ndimage.map_coordinates(f, sample_coords(dom, disp), order=order, mode="grid-wrap")


def fourier_warp(dom, f, disp):
    """Trigonometric interpolant at x + u(x) (gridops.py:51-75)."""
    shape, d = dom.shape, dom.ndim
    spec = scipy.fft.fftn(f) / float(np.prod(shape))
    coords = sample_coords(dom, disp)
    npts = int(np.prod(shape))
    phases = []
    for ax, n in enumerate(shape):
        fr = np.rint(np.fft.fftfreq(n, 1.0 / n)).astype(np.int64)
        x = coords[ax].reshape(npts) / n
        ph = np.exp(2j * np.pi * np.outer(x, fr))
        if n % 2 == 0:
            ph[:, n // 2] = np.cos(2.0 * np.pi * x * (n // 2))
        phases.append(ph)
    acc = np.tensordot(spec, phases[-1], axes=([d - 1], [1]))
    for ax in range(d - 2, -1, -1):
        acc = np.einsum("...kp,pk->...p", acc, phases[ax])
    return acc.real.reshape(shape)


def grid_grad(dom, f, mode="central"):  # gridops.py:78-100
    d = dom.ndim
    out = np.empty((d,) + dom.shape)
    if mode == "central":
        for ax, h in enumerate(dom.h):
            out[ax] = (np.roll(f, -1, axis=ax) - np.roll(f, 1, axis=ax)) / (2.0 * h)
        return out
    if mode == "spectral":
        spec = scipy.fft.fftn(f)
        for ax, n in enumerate(dom.shape):
            k = np.rint(np.fft.fftfreq(n, 1.0 / n)).astype(np.float64)
            if n % 2 == 0:
                k[n // 2] = 0.0
            out[ax] = scipy.fft.ifftn(spec * (2j * np.pi * _bcast(k, ax, d))).real
        return out
    raise ValueError(mode)


def jacobian_det(dom, disp):  # gridops.py:103-131
    d = dom.ndim
    J = np.empty((d, d) + dom.shape)
    for i in range(d):
        g = grid_grad(dom, disp[i])
        for j in range(d):
            J[i, j] = g[j] + (1.0 if i == j else 0.0)
    if d == 1:
        return J[0, 0].copy()
    if d == 2:
        return J[0, 0] * J[1, 1] - J[0, 1] * J[1, 0]
    a, b, c = J
    return (a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0])
            + a[2] * (b[0] * c[1] - b[1] * c[0]))


# ---------------------------------------------------------------------------
# objectives (objectives/base.py, state.py, deformation.py)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Problem:
    """Restates ``ProblemConfig`` (objectives/base.py:27-65)."""
    sigma2: float = 1.0
    gamma: int = 0
    n_time_steps: int = 10
    interp: str = "linear"
    image_grad: str = "central"
    quadrature: str = "trapezoid"
    cfl_limit: float = 0.5
    auto_refine: bool = True
    contraction: str = "transposed"


@dataclass
class Eval:
    """Restates ``Evaluation`` + the per-objective caches."""
    velocity: Flow
    energy: float
    reg_energy: float
    data_energy: float
    gradient: Flow
    warped_source: np.ndarray
    adjoint_end: np.ndarray
    substeps: int
    forward: np.ndarray
    extra: dict = field(default_factory=dict)


class OracleObjective:
    """Shared pipeline (objectives/base.py:92-188); ``kind`` selects the
    state (state.py) or deformation (deformation.py) adjoint."""

    def __init__(self, dom: Dom, source, target, cfg: Problem | None = None, kind="state"):
        self.dom, self.cfg, self.kind = dom, cfg or Problem(), kind
        self.source = np.ascontiguousarray(source, dtype=np.float64)
        self.target = np.ascontiguousarray(target, dtype=np.float64)
        if self.source.shape != dom.shape or self.target.shape != dom.shape:
            raise ValueError("images must be scalar fields on the domain grid")
        if not (np.all(np.isfinite(self.source)) and np.all(np.isfinite(self.target))):
            raise ValueError("images contain NaN or Inf")
        self._sg = None

    # base.py:112-118
    @property
    def source_gradient(self):
        if self._sg is None:
            self._sg = grid_grad(self.dom, self.source, self.cfg.image_grad)
        return self._sg

    def _warp(self, f, disp_grid):
        return warp(self.dom, f, disp_grid, self.cfg.interp)

    def _lam_end(self, m1):  # base.py:136-140
        lam = -(2.0 / self.cfg.sigma2) * (m1 - self.target)
        if not np.all(np.isfinite(lam)):
            raise ValueError("adjoint endpoint is not finite; sigma2 may be too small")
        return lam

    def reg_energy(self, v: Flow):  # base.py:142-151
        if v.stationary:
            return 0.5 * inner(helmholtz(self.dom, v.values[0]), v.values[0])
        w = time_weights(v.n_steps, self.cfg.quadrature)
        return 0.5 * sum(w[i] * inner(helmholtz(self.dom, v.values[i]), v.values[i])
                         for i in range(v.n_nodes))

    def data_energy(self, m1):  # base.py:153-155
        return grid_norm2(self.dom, m1 - self.target) / self.cfg.sigma2

    def assemble(self, v: Flow, data):  # base.py:157-179
        dom = self.dom
        free = self.cfg.gamma == 1
        if v.stationary:
            w = time_weights(v.n_steps, self.cfg.quadrature)
            g = helmholtz(dom, v.values[0]) + sum(w[i] * data[i] for i in range(v.n_nodes))
            if free:
                g = leray(dom, g)
            return v.like(g[None])
        out = np.empty_like(v.values)
        for i in range(v.n_nodes):
            g = helmholtz(dom, v.values[i]) + data[i]
            out[i] = leray(dom, g) if free else g
        return v.like(out)

    def substeps(self, v):
        return substeps_for(v, self.cfg.cfl_limit, self.cfg.auto_refine)

    def energy(self, v: Flow):  # base.py:183-188
        phi = forward_map(v, self.substeps(v))
        m1 = self._warp(self.source, include(self.dom, phi[-1], check=False))
        return self.reg_energy(v) + self.data_energy(m1)

    # -- gradient ------------------------------------------------------------
    def gradient(self, v: Flow) -> Eval:
        return self._grad_state(v) if self.kind == "state" else self._grad_def(v)

    def _grad_state(self, v):  # state.py:73-108
        dom = self.dom
        ns = self.substeps(v)
        phi = forward_map(v, ns)
        psi, vol = inverse_map_and_volume(v, ns)
        fwd = [include(dom, x, check=False) for x in phi]
        inv = [include(dom, x, check=False) for x in psi]
        volg = [include(dom, x, check=False) for x in vol]
        m = [self._warp(self.source, x) for x in fwd]
        lam1 = self._lam_end(m[-1])
        lam1_w = [self._warp(lam1, x) for x in inv]
        lam = [volg[i] * lam1_w[i] for i in range(len(volg))]
        gm = [grid_grad(dom, x, self.cfg.image_grad) for x in m]
        data = [project(dom, lam[i][None] * gm[i]) for i in range(len(lam))]
        g = self.assemble(v, data)
        er, ed = self.reg_energy(v), self.data_energy(m[-1])
        return Eval(v, er + ed, er, ed, g, m[-1], lam1, ns, phi,
                    dict(inverse=psi, volume=vol, fwd=fwd, inv=inv, volg=volg, m=m,
                         lam1_w=lam1_w, lam=lam, gm=gm))

    def _contract(self, phi_blk, rho):  # deformation.py:63-72
        return rho + conv_matvec(self.dom, jac(self.dom, phi_blk), rho,
                                 transpose=self.cfg.contraction == "transposed")

    def _grad_def(self, v):  # deformation.py:74-107
        dom = self.dom
        ns = self.substeps(v)
        phi = forward_map(v, ns)
        fwd = [include(dom, x, check=False) for x in phi]
        m1 = self._warp(self.source, fwd[-1])
        lam1 = self._lam_end(m1)
        gm1 = grid_grad(dom, m1, self.cfg.image_grad)
        sgw = np.stack([self._warp(self.source_gradient[a], fwd[-1]) for a in range(dom.ndim)])
        eg = sgw if self.cfg.contraction == "transposed" else gm1
        rho_end = project(dom, lam1[None] * eg)
        rho = momentum(v, rho_end, ns)
        data = [self._contract(phi[i], rho[i]) for i in range(v.n_nodes)]
        g = self.assemble(v, data)
        er, ed = self.reg_energy(v), self.data_energy(m1)
        return Eval(v, er + ed, er, ed, g, m1, lam1, ns, phi,
                    dict(fwd=fwd, gm1=gm1, sgw=sgw, rho=rho, rho_end=rho_end))

    # -- Hessian-vector products --------------------------------------------
    def hessian_vector(self, ev: Eval, w: Flow, gauss_newton=False) -> Flow:
        if self.kind == "state":
            return self._hvp_state(ev, w, gauss_newton)
        return self._hvp_def(ev, w, gauss_newton)

    def _hvp_state(self, ev, w, gn):  # state.py:110-154
        dom, v, x = self.dom, ev.velocity, ev.extra
        if gn:
            dphi = state_tangents(v, w, ev.substeps, with_volume=False, with_inverse=False)[0]
            dpsi = dvol = None
        else:
            dphi, dpsi, dvol = state_tangents(v, w, ev.substeps, with_volume=True)
        sgw = x.get("sgw_nodes")
        if sgw is None:  # state.py:38-49 (lazy)
            sgw = [np.stack([self._warp(self.source_gradient[a], f) for a in range(dom.ndim)])
                   for f in x["fwd"]]
            x["sgw_nodes"] = sgw
        dphi1 = include(dom, dphi[-1], check=False)
        dlam1 = -(2.0 / self.cfg.sigma2) * np.einsum("a...,a...->...", sgw[-1], dphi1)
        data = []
        if gn:
            for i in range(v.n_nodes):
                dlam = x["volg"][i] * self._warp(dlam1, x["inv"][i])
                data.append(project(dom, dlam[None] * x["gm"][i]))
        else:
            agw = x.get("agw_nodes")
            if agw is None:  # state.py:51-62 (lazy)
                ga = grid_grad(dom, ev.adjoint_end, self.cfg.image_grad)
                agw = [np.stack([self._warp(ga[a], f) for a in range(dom.ndim)]) for f in x["inv"]]
                x["agw_nodes"] = agw
            for i in range(v.n_nodes):
                dphi_g = include(dom, dphi[i], check=False)
                dpsi_g = include(dom, dpsi[i], check=False)
                dvol_g = include(dom, dvol[i], check=False)
                dm = np.einsum("a...,a...->...", sgw[i], dphi_g)
                dlam = (dvol_g * x["lam1_w"][i]
                        + x["volg"][i] * np.einsum("a...,a...->...", agw[i], dpsi_g)
                        + x["volg"][i] * self._warp(dlam1, x["inv"][i]))
                term = dlam[None] * x["gm"][i] + x["lam"][i][None] * grid_grad(
                    dom, dm, self.cfg.image_grad)
                data.append(project(dom, term))
        return self.assemble(w, data)

    def _hvp_def(self, ev, w, gn):  # deformation.py:109-153
        dom, v, x = self.dom, ev.velocity, ev.extra
        tr = self.cfg.contraction == "transposed"
        dphi = state_tangents(v, w, ev.substeps, with_volume=False, with_inverse=False)[0]
        dphi1 = include(dom, dphi[-1], check=False)
        dlam1 = -(2.0 / self.cfg.sigma2) * np.einsum("a...,a...->...", x["sgw"], dphi1)
        eg = x["sgw"] if tr else x["gm1"]
        term = dlam1[None] * eg
        if not gn:
            if tr:
                H = x.get("shess")
                if H is None:  # deformation.py:40-57 (lazy)
                    d = dom.ndim
                    hs = np.empty((d, d) + dom.shape)
                    for a in range(d):
                        ga = grid_grad(dom, self.source_gradient[a], self.cfg.image_grad)
                        for b in range(d):
                            hs[a, b] = ga[b]
                    H = np.empty_like(hs)
                    for a in range(d):
                        for b in range(d):
                            H[a, b] = self._warp(hs[a, b], x["fwd"][-1])
                    x["shess"] = H
                term = term + ev.adjoint_end[None] * np.einsum("ab...,b...->a...", H, dphi1)
            else:
                dm1 = np.einsum("a...,a...->...", x["sgw"], dphi1)
                term = term + ev.adjoint_end[None] * grid_grad(dom, dm1, self.cfg.image_grad)
        drho_end = project(dom, term)
        rho, drho = momentum_tangent(v, w, x["rho_end"], drho_end, ev.substeps, gauss_newton=gn)
        data = []
        for i in range(v.n_nodes):
            node = self._contract(ev.forward[i], drho[i])
            if not gn:
                node = node + conv_matvec(dom, jac(dom, dphi[i]), rho[i], transpose=tr)
            data.append(node)
        return self.assemble(w, data)


# ---------------------------------------------------------------------------
# solver (solver.py:26-243)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SolverCfg:
    """Restates ``SolverConfig`` (solver.py:26-47)."""
    method: str = "gauss_newton"
    max_outer: int = 50
    grad_tol: float = 0.01
    pcg_tol: float = 0.1
    pcg_max_iter: int = 10
    ls_shrink: float = 0.5
    ls_c1: float = 1e-4
    step0: float = 1.0
    max_halvings: int = 20
    eisenstat_walker: bool = False


@dataclass
class Record:  # solver.py:50-59
    outer: int
    energy: float
    mse_rel: float
    grad_rel: float
    pcg_iters: int
    step: float
    negative_curvature: bool
    wall_time: float


@dataclass
class Result:  # solver.py:62-71
    velocity: Flow
    records: list = field(default_factory=list)
    status: str = "running"
    final_grad_rel: float = float("nan")
    final_mse_rel: float = float("nan")
    negative_curvature_events: int = 0
    total_pcg_iters: int = 0
    evaluation: object = None
    counters: dict = field(default_factory=dict)


def pcg(apply_h, g: Flow, cfg: SolverCfg, precond, rule):  # solver.py:88-126
    def ip(a, b):
        return flow_inner(a, b, rule)
    if math.sqrt(ip(g, g)) == 0.0:
        return g.like(g.values * 0.0), 0, False
    x = g.like(g.values * 0.0)
    r = g.like(g.values.copy())
    z = precond(r)
    p = z.like(z.values.copy())
    rz = ip(r, z)
    res0 = math.sqrt(max(rz, 0.0))
    for it in range(cfg.pcg_max_iter):
        hp = apply_h(p)
        php = ip(p, hp)
        if not np.isfinite(php):
            raise FloatingPointError("PCG encountered a non-finite curvature value")
        if php <= 0.0:
            return (z if it == 0 else x), it, True
        a = rz / php
        x = x.like(x.values + a * p.values)
        r = r.like(r.values - a * hp.values)
        z = precond(r)
        rzn = ip(r, z)
        if not np.isfinite(rzn):
            raise FloatingPointError("PCG encountered a non-finite residual")
        if math.sqrt(max(rzn, 0.0)) <= cfg.pcg_tol * res0:
            return x, it + 1, False
        p = p.like(z.values + (rzn / rz) * p.values)
        rz = rzn
    return x, cfg.pcg_max_iter, False


def minimize(obj: OracleObjective, v0: Flow, cfg: SolverCfg | None = None, mse_reference=None):
    """Outer GN/Newton/GD loop with Armijo backtracking (solver.py:129-243)."""
    cfg = cfg or SolverCfg()
    dom = obj.dom
    rule = obj.cfg.quadrature
    free = obj.cfg.gamma == 1
    counters = dict(gradient=0, hvp=0, energy=0, substeps=[])

    def pfree(f):
        return f.map_nodes(lambda c: leray(dom, c)) if free else f

    def precond(f):
        return pfree(f.map_nodes(lambda c: inv_helmholtz(dom, c)))

    if mse_reference is None:
        mse_reference = grid_norm2(dom, obj.source - obj.target)
    v = pfree(v0.like(v0.values.copy()))
    res = Result(velocity=v, counters=counters)
    t0 = time.perf_counter()
    g0 = None
    best_v, best_e = v, np.inf
    tol = cfg.pcg_tol
    prev = None
    for outer in range(cfg.max_outer):
        ev = obj.gradient(v)
        counters["gradient"] += 1
        counters["substeps"].append(ev.substeps)
        g = ev.gradient
        if g0 is None:
            g0 = g.max_speed()
        grel = 0.0 if g0 == 0.0 else g.max_speed() / g0
        mse = (100.0 * grid_norm2(dom, ev.warped_source - obj.target) / mse_reference
               if mse_reference > 0 else 0.0)
        if ev.energy < best_e:
            best_v, best_e = v, ev.energy
        if grel <= cfg.grad_tol:
            res.records.append(Record(outer, ev.energy, mse, grel, 0, 0.0, False,
                                      time.perf_counter() - t0))
            res.status, res.velocity, res.evaluation = "converged", v, ev
            break
        if cfg.method == "gradient_descent":
            step, its, neg = precond(g), 0, False
        else:
            gn = cfg.method == "gauss_newton"
            if cfg.eisenstat_walker and prev is not None:
                ratio = g.max_speed() / prev
                tol = float(min(cfg.pcg_tol, max(1e-4, ratio * ratio)))
            lcfg = cfg if tol == cfg.pcg_tol else replace(cfg, pcg_tol=tol)

            def apply_h(f, ev=ev, gn=gn):
                counters["hvp"] += 1
                return pfree(obj.hessian_vector(ev, f, gn))

            step, its, neg = pcg(apply_h, g, lcfg, precond, rule)
            if neg:
                res.negative_curvature_events += 1
        res.total_pcg_iters += its
        slope = flow_inner(g, step, rule)
        if slope <= 0.0:
            step = precond(g)
            slope = flow_inner(g, step, rule)
        eps = cfg.step0
        ok = False
        for _ in range(cfg.max_halvings):
            trial = pfree(v.like(v.values - eps * step.values))
            counters["energy"] += 1
            if obj.energy(trial) <= ev.energy - cfg.ls_c1 * eps * slope:
                ok = True
                break
            eps *= cfg.ls_shrink
        prev = g.max_speed()
        res.records.append(Record(outer, ev.energy, mse, grel, its, eps if ok else 0.0, neg,
                                  time.perf_counter() - t0))
        if not ok:
            res.status, res.velocity = "stalled", best_v
            break
        v = trial
        res.velocity = v
    else:
        res.status, res.velocity = "budget_exhausted", v
    if res.evaluation is None:
        res.evaluation = obj.gradient(res.velocity)
    fin = res.evaluation
    res.final_grad_rel = fin.gradient.max_speed() / (g0 or 1.0) if (g0 or 1.0) != 0 else 0.0
    res.final_mse_rel = (100.0 * grid_norm2(dom, fin.warped_source - obj.target) / mse_reference
                         if mse_reference > 0 else 0.0)
    return res


# ---------------------------------------------------------------------------
# synthetic inputs (tests/helpers.py:9-129, synthesis.py:20-60)
# ---------------------------------------------------------------------------

def random_vector_block(dom, rng, scale=1.0):  # helpers.py:16-19
    sh = (dom.ndim,) + dom.block
    c = rng.standard_normal(sh) + 1j * rng.standard_normal(sh)
    return symmetrize(scale * c, dom.ndim)


def random_scalar_block(dom, rng, scale=1.0):  # helpers.py:9-13
    c = rng.standard_normal(dom.block) + 1j * rng.standard_normal(dom.block)
    return symmetrize(scale * c, dom.ndim)


def smooth_vector_block(dom, rng, scale=1.0, decay=1.5):  # helpers.py:22-37
    c = random_vector_block(dom, rng)
    k2 = np.zeros(dom.block)
    for ax, m in enumerate(dom.block):
        k2 = k2 + _bcast(freqs_of(m).astype(float) ** 2, ax, dom.ndim)
    c = c / (1.0 + k2) ** decay
    return c * (scale / max_abs(dom, c))


def band_image(dom, rng, decay=3.0, amp=1.0):  # helpers.py:93-100
    c = smooth_vector_block(dom, rng, 1.0, decay=decay)[0]
    img = include(dom, c)
    img = img - img.min()
    return amp * img / img.max()


def smooth_flow(dom, rng, amp=0.04, n_steps=32, stationary=True, gamma=0, decay=3.0):
    """helpers.py:103-120."""
    if stationary:
        vals = smooth_vector_block(dom, rng, amp, decay=decay)[None]
    else:
        a = smooth_vector_block(dom, rng, amp, decay=decay)
        b = smooth_vector_block(dom, rng, amp, decay=decay)
        c = smooth_vector_block(dom, rng, amp, decay=decay)
        t = np.arange(n_steps + 1) / n_steps
        sh = (-1,) + (1,) * (dom.ndim + 1)
        vals = a[None] + b[None] * np.sin(np.pi * t).reshape(sh) + c[None] * (t ** 2).reshape(sh)
    f = Flow(dom, vals, n_steps, stationary)
    return f.map_nodes(lambda x: leray(dom, x)) if gamma else f


def periodic_bump(mesh, center, sharpness):  # synthesis.py:20-25
    out = np.ones_like(mesh[0])
    for x, c in zip(mesh, center):
        out = out * np.exp(sharpness * (np.cos(2 * np.pi * (x - c)) - 1.0))
    return out


def mesh(shape):  # synthesis.py:15-17
    return np.meshgrid(*[np.arange(n) / n for n in shape], indexing="ij")


def translation_pair(size=64, seed=0, shift=0.1):
    """2-D ``translation`` pair (synthesis.py:37-60)."""
    m = mesh((size, size))
    rng = np.random.default_rng(seed)
    jit = 0.02 * rng.standard_normal(2)
    c = np.array([0.5, 0.5]) + jit
    return periodic_bump(m, c, 24.0), periodic_bump(m, c + np.array([shift, 0.0]), 24.0)


def blob_pair_3d(n, seed=0, n_blobs=6, k_def=4, amp_vox=3.0):
    """Seeded 3-D synthetic pair for configs 2-4 (new; the reference's pairs are
    2-D only, synthesis.py:51).  Source: sum of periodic bumps; target: source
    warped (cubic) by a smooth band-K_def displacement of ~amp_vox voxels."""
    shape = (n, n, n)
    m = mesh(shape)
    rng = np.random.default_rng(seed)
    src = np.zeros(shape)
    for _ in range(n_blobs):
        c = 0.3 + 0.4 * rng.random(3)
        src += (0.5 + 0.5 * rng.random()) * periodic_bump(m, c, 8.0 + 16.0 * rng.random())
    src /= src.max()
    ddom = Dom(shape, (k_def,) * 3)
    disp = include(ddom, smooth_vector_block(ddom, rng, amp_vox / n, decay=2.0))
    tgt = warp(ddom, src, disp, "cubic")
    return src, tgt
