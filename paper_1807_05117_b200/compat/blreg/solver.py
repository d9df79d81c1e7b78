"""Solver (reference ``solver.py``) over host flows: the PCG vector updates,
inner products, gradients and Hessian products run on the device."""

from paper_1807_05117_b200 import solver as _sv
from paper_1807_05117_b200.solver import IterationRecord, SolverConfig  # noqa: F401

from .transport import TimeFlow, _d


def relative_gradient_norm(gradient, initial, initial_norm=None) -> float:
    return _sv.relative_gradient_norm(_d(gradient), _d(initial) if initial is not None else None, initial_norm)


def pcg_solve(apply_h, g, cfg, apply_precond, quadrature: str):
    """Host callables are wrapped so they see (and return) host flows."""
    def wrap(fn):
        return lambda f: fn(TimeFlow.from_device(f)).device()
    x, it, neg = _sv.pcg_solve(wrap(apply_h), g.device(), cfg, wrap(apply_precond), quadrature)
    return TimeFlow.from_device(x), it, neg


class SolveResult:
    def __init__(self, res, objective):
        from .objectives import Evaluation

        self._r = res
        self.records = res.records
        self.status = res.status
        self.final_grad_rel = res.final_grad_rel
        self.final_mse_rel = res.final_mse_rel
        self.negative_curvature_events = res.negative_curvature_events
        self.total_pcg_iters = res.total_pcg_iters
        self.velocity = TimeFlow.from_device(res.velocity)
        self.evaluation = (Evaluation(objective, res.evaluation, self.velocity)
                           if res.evaluation is not None else None)


def minimize(objective, v0, cfg=None, mse_reference=None):
    return SolveResult(_sv.minimize(objective._obj, v0.device(), cfg, mse_reference), objective)
