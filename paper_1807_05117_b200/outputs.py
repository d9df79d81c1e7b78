"""Post-registration outputs: quality metrics on the device and the BLVOL
volume file format (``blreg/metrics.py``, ``blreg/volio.py``).

Metrics take device (or host) arrays and reduce on the GPU; ``write_volume``
produces files byte-identical to the reference writer (ASCII header +
little-endian float32 payload, component axis first for vector fields).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

MAGIC = b"BLVOL 1"


def _t(x):
    return x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x))


def mse_rel(warped, source, target) -> float:
    """``100 * ||warped - target||^2 / ||source - target||^2`` (metrics.py:8-19)."""
    w, s, t = _t(warped).double(), _t(source).double(), _t(target).double()
    dev = w.device
    s, t = s.to(dev), t.to(dev)
    denom = float(((s - t) ** 2).sum())
    if denom == 0.0:
        return 0.0
    return 100.0 * float(((w - t) ** 2).sum()) / denom


def dice(a, b, label: int = 1) -> float:
    """``2|A & B| / (|A| + |B|)`` for one label; 1 if both empty (metrics.py:22-30)."""
    ta, tb = _t(a), _t(b)
    if ta.shape != tb.shape:
        raise ValueError("label volumes must share a grid")
    ma, mb = ta == label, tb.to(ta.device) == label
    total = int(ma.sum()) + int(mb.sum())
    if total == 0:
        return 1.0
    return 2.0 * int((ma & mb).sum()) / total


def jacobian_extrema(det) -> tuple:
    t = _t(det)
    return float(t.min()), float(t.max())


# ---------------------------------------------------------------------------
# BLVOL files (volio.py:16-99)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class VolumeHeader:
    dims: tuple
    spacing: tuple
    components: int = 1
    dtype: str = "float32"
    byteorder: str = "little"
    layout: str = "axis-major"


class VolumeFormatError(ValueError):
    pass


def _host(values) -> np.ndarray:
    if isinstance(values, torch.Tensor):
        return values.detach().cpu().numpy()
    return np.asarray(values)


def write_volume(path, values, spacing=None) -> None:
    """Write a scalar ``(*dims)`` or vector ``(d, *dims)`` field."""
    arr = _host(values)
    if arr.ndim < 1:
        raise VolumeFormatError("volume payload must be an array")
    vector = arr.ndim >= 2 and arr.shape[0] == arr.ndim - 1
    comps, dims = (arr.shape[0], arr.shape[1:]) if vector else (1, arr.shape)
    spacing = tuple(1.0 / n for n in dims) if spacing is None else tuple(spacing)
    if len(spacing) != len(dims):
        raise VolumeFormatError("spacing must have one entry per axis")
    header = [MAGIC.decode(), "dims: " + " ".join(str(int(n)) for n in dims),
              "spacing: " + " ".join(repr(float(s)) for s in spacing), f"components: {comps}",
              "dtype: float32", "byteorder: little", "layout: axis-major", "end-header"]
    with open(path, "wb") as fh:
        fh.write(("\n".join(header) + "\n").encode("ascii"))
        fh.write(np.ascontiguousarray(arr, dtype="<f4").tobytes(order="C"))


def read_volume(path):
    """Returns (float32 values, VolumeHeader)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    end = blob.find(b"\nend-header\n")
    if not blob.startswith(MAGIC + b"\n"):
        raise VolumeFormatError(f"{path}: not a volume file")
    if end < 0:
        raise VolumeFormatError(f"{path}: truncated header")
    fields = {}
    for line in blob[len(MAGIC) + 1:end].split(b"\n"):
        key, sep, val = line.decode("ascii").partition(":")
        if not sep:
            raise VolumeFormatError(f"{path}: malformed header line {line!r}")
        fields[key.strip()] = val.strip()
    try:
        dims = tuple(int(t) for t in fields["dims"].split())
        spacing = tuple(float(t) for t in fields["spacing"].split())
        comps = int(fields.get("components", "1"))
    except (KeyError, ValueError) as exc:
        raise VolumeFormatError(f"{path}: invalid header fields") from exc
    if fields.get("dtype", "float32") != "float32" or fields.get("byteorder", "little") != "little":
        raise VolumeFormatError(f"{path}: unsupported payload encoding")
    payload = blob[end + len(b"\nend-header\n"):]
    count = int(np.prod(dims)) * comps
    if len(payload) != 4 * count:
        raise VolumeFormatError(f"{path}: payload holds {len(payload)} bytes, expected {4 * count}")
    vals = np.frombuffer(payload, dtype="<f4").copy()
    return vals.reshape(dims if comps == 1 else (comps,) + dims), VolumeHeader(dims, spacing, comps)
