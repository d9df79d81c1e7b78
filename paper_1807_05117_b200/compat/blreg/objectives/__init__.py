"""Objectives (reference ``objectives/``) with host (numpy) inputs and
results; energies, gradients and Hessian-vector products run on the B200."""

from paper_1807_05117_b200 import objectives as _o
from paper_1807_05117_b200.objectives import ProblemConfig  # noqa: F401

from .._conv import host
from ..transport import TimeFlow, TrajectoryCache

__all__ = ["Evaluation", "ProblemConfig", "StateObjective", "DeformationObjective"]


class Evaluation:
    """Host view of a device evaluation (reference ``objectives/base.py:68-89``):
    scalars directly, arrays copied to host on first access."""

    def __init__(self, objective, ev, velocity):
        self.objective = objective
        self._ev = ev
        self.velocity = velocity
        self.energy = ev.energy
        self.reg_energy = ev.reg_energy
        self.data_energy = ev.data_energy
        self.cache = TrajectoryCache(ev.cache, velocity)
        self._h = {}

    def _get(self, name, fn):
        if name not in self._h:
            self._h[name] = fn()
        return self._h[name]

    gradient = property(lambda self: self._get("gradient", lambda: TimeFlow.from_device(self._ev.gradient)))
    warped_source = property(lambda self: self._get("warped_source", lambda: host(self._ev.warped_source)))
    adjoint_end = property(lambda self: self._get("adjoint_end", lambda: host(self._ev.adjoint_end)))

    def hessian_vector(self, direction, gauss_newton: bool = False):
        return self.objective.hessian_vector(self, direction, gauss_newton=gauss_newton)


class _Objective:
    _cls = None

    def __init__(self, domain, source, target, config=None):
        self._obj = self._cls(domain, source, target, config)
        self.domain = domain
        self.config = self._obj.config
        self.source = self._obj.source
        self.target = self._obj.target

    def energy(self, v) -> float:
        return self._obj.energy(v.device())

    def gradient(self, v) -> Evaluation:
        return Evaluation(self, self._obj.gradient(v.device()), v)

    def hessian_vector(self, evaluation: Evaluation, direction, gauss_newton: bool = False):
        evaluation.cache.assert_matches(evaluation.velocity)
        evaluation.velocity._check_compatible(direction)
        hv = self._obj.hessian_vector(evaluation._ev, direction.device(), gauss_newton=gauss_newton)
        return TimeFlow.from_device(hv)


class StateObjective(_Objective):
    _cls = _o.StateObjective


class DeformationObjective(_Objective):
    _cls = _o.DeformationObjective
