"""Computational domain and its device context.

``Domain`` keeps the reference's constructor and validation
(``blreg/domain.py:19-63``) and adds three B200 options:

* ``pad``  — pad-grid points per axis for truncated convolutions.  The
  reference uses ``next_fast_len(4K+1)`` (``spectral.py:142-145``); any
  ``P >= 3K+1`` gives the exact truncated convolution because every pad-grid
  product is bilinear in K-band fields, so the default is the smallest
  engine length >= 3K+1 (e.g. 100 instead of 132 at K=32, 2.3x fewer points).
* ``dtype`` — ``"float64"`` (parity mode, complex128 blocks) or ``"float32"``.
* ``device`` — CUDA device index.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np
import torch

from . import _lib

_TWO_PI = 2.0 * np.pi


def smooth_size(n: int, primes=(2, 3, 5, 7)) -> int:
    """Smallest m >= n whose prime factors are all in ``primes``."""
    m = max(int(n), 1)
    while True:
        r = m
        for p in primes:
            while r % p == 0:
                r //= p
        if r == 1:
            return m
        m += 1


# Pad lengths the fused sm_100a pad engine implements (L = R1*R2 warp FFTs,
# csrc/blr_fft.cuh BLR_FOR_EACH_L); other 7-smooth pads run the cuFFT path.
ENGINE_PADS = (10, 14, 16, 20, 25, 28, 32, 40, 49, 50, 64, 100, 196)


def default_pad(bandwidth) -> tuple:
    """Smallest engine pad >= 3K+1 per axis (exact truncated convolution),
    else the smallest 7-smooth size >= 3K+1."""
    out = []
    for k in bandwidth:
        need = 3 * k + 1
        fast = [p for p in ENGINE_PADS if p >= need]
        out.append(fast[0] if fast else smooth_size(need))
    return tuple(out)


@dataclass(frozen=True)
class Domain:
    """Grid sizes, frequency bounds and metric parameters (domain.py:19-97)."""

    shape: tuple
    bandwidth: tuple
    alpha: float = 0.02
    order: int = 2
    symbol: str = "discrete"
    pad: tuple | None = None
    dtype: str = "float64"
    device: int = 0

    def __post_init__(self):
        shape = tuple(int(n) for n in self.shape)
        bandwidth = tuple(int(k) for k in self.bandwidth)
        object.__setattr__(self, "shape", shape)
        object.__setattr__(self, "bandwidth", bandwidth)
        if len(shape) not in (1, 2, 3):
            raise ValueError(f"only 1-, 2- or 3-dimensional grids are supported, got {shape}")
        if len(bandwidth) != len(shape):
            raise ValueError("bandwidth must have one entry per grid axis")
        for n, k in zip(shape, bandwidth):
            if n < 2:
                raise ValueError(f"grid size {n} is too small")
            if not 1 <= k <= n // 2:
                raise ValueError(f"bandwidth {k} outside [1, {n // 2}] for grid size {n}")
        if not self.alpha > 0:
            raise ValueError("alpha must be positive")
        if not (isinstance(self.order, (int, np.integer)) and self.order >= 1):
            raise ValueError("order must be an integer >= 1")
        if self.symbol not in ("discrete", "continuous"):
            raise ValueError(f"unknown symbol {self.symbol!r}")
        pad = default_pad(bandwidth) if self.pad is None else tuple(int(p) for p in self.pad)
        if len(pad) != len(shape) or any(p < 3 * k + 1 for p, k in zip(pad, bandwidth)):
            raise ValueError(f"pad grid {pad} must have at least 3K+1 points per axis")
        object.__setattr__(self, "pad", pad)
        if self.dtype not in ("float64", "float32"):
            raise ValueError("dtype must be 'float64' or 'float32'")

    # -- reference API -------------------------------------------------------
    @property
    def ndim(self) -> int:
        return len(self.shape)

    @property
    def spacing(self) -> tuple:
        return tuple(1.0 / n for n in self.shape)

    @property
    def block_shape(self) -> tuple:
        return tuple(2 * k + 1 for k in self.bandwidth)

    @property
    def cell_volume(self) -> float:
        return float(np.prod(self.spacing))

    def frequencies(self):
        return tuple(np.rint(np.fft.fftfreq(m, 1.0 / m)).astype(np.int64) for m in self.block_shape)

    def zero_scalar(self):
        return torch.zeros(self.block_shape, dtype=self.cdtype, device=self.torch_device)

    def zero_vector(self):
        return torch.zeros((self.ndim,) + self.block_shape, dtype=self.cdtype, device=self.torch_device)

    # -- device helpers --------------------------------------------------------
    @property
    def rdtype(self):
        return torch.float64 if self.dtype == "float64" else torch.float32

    @property
    def cdtype(self):
        return torch.complex128 if self.dtype == "float64" else torch.complex64

    @property
    def torch_device(self):
        return torch.device("cuda", self.device)

    @property
    def n_band(self) -> int:
        return int(np.prod(self.block_shape))

    @property
    def n_grid(self) -> int:
        return int(np.prod(self.shape))

    @property
    def n_pad(self) -> int:
        return int(np.prod(self.pad))

    def ctx(self) -> "Context":
        return _context(self)

    def with_dtype(self, dtype: str) -> "Domain":
        return Domain(self.shape, self.bandwidth, self.alpha, self.order, self.symbol, self.pad,
                      dtype, self.device)

    def compatible(self, other: "Domain") -> bool:
        return self == other


def symbol_terms(domain: Domain) -> np.ndarray:
    """alpha-free per-axis metric symbol terms (spectral.py:242-257), concatenated."""
    out = []
    for f, n in zip(domain.frequencies(), domain.shape):
        if domain.symbol == "discrete":
            term = 2.0 * n * n * (1.0 - np.cos(_TWO_PI * f / n))
        else:
            term = (_TWO_PI * f) ** 2
        out.append(np.asarray(term, dtype=np.float64))
    return np.concatenate(out)


class Context:
    """Device contexts (``blr_ctx``: cuFFT plans, engine scratch) for a domain.

    Thread / stream safety (reference contract ``objectives/base.py:69-72``:
    ``hessian_vector`` may be called concurrently on one evaluation): every
    (host thread, torch stream) pair gets its own ``blr_ctx``, created on first
    use with its stream fixed, so no scratch buffer and no host-side state is
    ever shared between two threads or between two streams.  Work issued by one
    thread on one stream is stream-ordered, so reusing that handle's scratch
    from call to call is safe.
    """

    def __init__(self, domain: Domain):
        if not torch.cuda.is_available():
            raise _lib.CudaExtensionMissing("no CUDA device: the B200 path has no CPU fallback")
        self.domain = domain
        self.lib = _lib.load()
        self._handles = {}  # (thread id, stream) -> blr_ctx*
        self.lock = threading.Lock()

    def _create(self, stream: int):
        d = self.domain
        h = C.c_void_p()
        tab, keep = _lib.double_array(symbol_terms(d))
        with torch.cuda.device(d.device):
            _lib.check(self.lib.blr_ctx_create(
                C.byref(h), d.ndim, _lib.int_array(d.shape), _lib.int_array(d.bandwidth),
                _lib.int_array(d.pad), float(d.alpha), int(d.order), tab,
                0 if d.dtype == "float64" else 1, int(d.device)), "blr_ctx_create")
            _lib.check(self.lib.blr_set_stream(h, C.c_void_p(stream)), "blr_set_stream")
        del keep
        return h

    def bind(self):
        """The handle for the calling thread on its current torch stream of
        ``domain.device``.  Entry points make the context's device current
        themselves (``blr_capi.cu`` DISPATCH), so callers need not."""
        s = torch.cuda.current_stream(self.domain.device).cuda_stream
        key = (threading.get_ident(), s)
        h = self._handles.get(key)
        if h is None:
            with self.lock:
                h = self._handles.get(key)
                if h is None:
                    h = self._create(s)
                    self._handles[key] = h
        return h

    @property
    def n_handles(self) -> int:
        return len(self._handles)

    def __del__(self):
        try:
            for h in self._handles.values():
                self.lib.blr_ctx_destroy(h)
        except Exception:
            pass


_ctx_lock = threading.Lock()


@lru_cache(maxsize=None)
def _context_cached(domain: Domain) -> Context:
    return Context(domain)


def _context(domain: Domain) -> Context:
    with _ctx_lock:
        return _context_cached(domain)
