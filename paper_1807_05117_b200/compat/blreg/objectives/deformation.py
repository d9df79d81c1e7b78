from . import *  # noqa: F401,F403
from . import Evaluation, DeformationObjective, ProblemConfig, StateObjective  # noqa: F401
