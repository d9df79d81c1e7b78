"""``Domain`` (reference ``domain.py:19-97``) with host (numpy) zero blocks."""

from dataclasses import dataclass

import numpy as np

from paper_1807_05117_b200.domain import Domain as _DeviceDomain


@dataclass(frozen=True)
class Domain(_DeviceDomain):
    """The device domain; ``zero_scalar`` / ``zero_vector`` return numpy blocks."""

    def zero_scalar(self) -> np.ndarray:
        return np.zeros(self.block_shape, dtype=np.complex128)

    def zero_vector(self) -> np.ndarray:
        return np.zeros((self.ndim,) + self.block_shape, dtype=np.complex128)


def _frequencies(block_shape):
    return tuple(np.rint(np.fft.fftfreq(m, 1.0 / m)).astype(np.int64) for m in block_shape)
