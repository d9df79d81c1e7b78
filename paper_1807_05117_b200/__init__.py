"""B200-native (sm_100a) Gauss-Newton-Krylov hot path of band-limited
PDE-constrained LDDMM (arXiv 1807.05117), API-compatible with the reference
package ``blreg``.

Host API (Python, mirrors the reference): ``Domain``, ``TimeFlow``,
``ProblemConfig``, ``StateObjective`` / ``DeformationObjective`` (``energy``,
``gradient``, ``Evaluation.hessian_vector``), ``pcg_solve``, ``minimize``.
Compute: the C-ABI shared library ``_lib/libblreg_b200.so``
(``include/blreg_b200.h``) — hand-written CUDA kernels + cuFFT, no CPU
fallback.
"""

from .domain import Domain
from .objectives import DeformationObjective, ProblemConfig, StateObjective
from .solver import SolverConfig, minimize, pcg_solve, relative_gradient_norm
from .transport import CFLViolation, TimeFlow, flow_inner, time_weights

__version__ = "0.1.0"

__all__ = [
    "Domain",
    "TimeFlow",
    "ProblemConfig",
    "StateObjective",
    "DeformationObjective",
    "SolverConfig",
    "minimize",
    "pcg_solve",
    "relative_gradient_norm",
    "flow_inner",
    "time_weights",
    "CFLViolation",
    "__version__",
]
