"""INI run configuration (reference ``runconfig.py:17-186``).

Sections ``[domain]``, ``[problem]``, ``[optimizer]``, ``[run]`` map onto
``Domain``, ``ProblemConfig``, ``SolverConfig`` and the run's inputs/outputs.
The schema below is the single source of truth: unknown sections' keys are
rejected (typos fail loudly), values are parsed by type, and every setting
not given takes the config dataclasses' own default, so
``effective_settings`` echoes the complete configuration into each report.
B200 additions in ``[domain]``: ``pad`` and ``dtype``.
"""

from __future__ import annotations

import configparser
from dataclasses import dataclass, fields

from ..domain import Domain
from ..objectives import ProblemConfig
from ..solver import SolverConfig


class ConfigError(ValueError):
    """Malformed or inconsistent run configuration."""


_TRUE = {"true", "1", "yes", "on"}
_FALSE = {"false", "0", "no", "off"}


def _bool(raw: str) -> bool:
    r = raw.lower()
    if r in _TRUE:
        return True
    if r in _FALSE:
        return False
    raise ValueError(raw)


def _ints(raw: str) -> tuple:
    return tuple(int(t) for t in raw.split())


_CASTS = {int: int, float: float, str: str, bool: _bool}


def _dataclass_schema(cls) -> dict:
    return {f.name: (_CASTS[f.type if not isinstance(f.type, str) else eval(f.type)], f.default)
            for f in fields(cls)}


# section -> key -> (parser, default)
SCHEMA = {
    "domain": {"shape": (_ints, None), "bandwidth": (_ints, None), "alpha": (float, 0.02),
               "order": (int, 2), "symbol": (str, "discrete"), "pad": (_ints, None),
               "dtype": (str, "float64")},
    "problem": {"objective": (str, "state"), "mode": (str, "stationary"),
                **_dataclass_schema(ProblemConfig)},
    "optimizer": _dataclass_schema(SolverConfig),
    "run": {"source": (str, ""), "target": (str, ""), "source_labels": (str, ""),
            "target_labels": (str, ""), "output_dir": (str, "out"), "seed": (int, 0)},
}


@dataclass(frozen=True)
class RunConfig:
    problem: ProblemConfig
    solver: SolverConfig
    objective: str
    mode: str
    shape: tuple | None
    bandwidth: tuple | None
    alpha: float
    order: int
    symbol: str
    pad: tuple | None
    dtype: str
    source: str
    target: str
    source_labels: str
    target_labels: str
    output_dir: str
    seed: int

    @property
    def domain(self) -> Domain | None:
        return self.domain_for(self.shape) if self.shape is not None else None

    def domain_for(self, shape: tuple) -> Domain:
        shape = tuple(int(n) for n in shape)
        if self.shape is not None and tuple(self.shape) != shape:
            raise ConfigError(f"configured grid {tuple(self.shape)} does not match volume {shape}")
        if self.bandwidth is None:
            raise ConfigError("bandwidth must be set in [domain]")
        bw = self.bandwidth * len(shape) if len(self.bandwidth) == 1 else self.bandwidth
        pad = None
        if self.pad is not None:
            pad = self.pad * len(shape) if len(self.pad) == 1 else self.pad
        try:
            return Domain(shape=shape, bandwidth=bw, alpha=self.alpha, order=self.order, symbol=self.symbol,
                          pad=pad, dtype=self.dtype)
        except ValueError as exc:
            raise ConfigError(str(exc)) from exc


def parse_sections(parser: configparser.ConfigParser) -> dict:
    values = {}
    for section, keys in SCHEMA.items():
        sec = parser[section] if parser.has_section(section) else {}
        unknown = sorted(set(sec) - set(keys))
        if unknown:
            raise ConfigError(f"unknown keys in [{section}]: {unknown}")
        for key, (cast, default) in keys.items():
            if key in sec:
                raw = sec[key].strip()
                try:
                    values[(section, key)] = cast(raw)
                except (KeyError, ValueError) as exc:
                    raise ConfigError(f"invalid value {raw!r} for {key}") from exc
            else:
                values[(section, key)] = default
    extra = sorted(set(parser.sections()) - set(SCHEMA))
    if extra:
        raise ConfigError(f"unknown sections: {extra}")
    return values


def load_config(path: str) -> RunConfig:
    parser = configparser.ConfigParser(inline_comment_prefixes=("#", ";"))
    if not parser.read(path):
        raise ConfigError(f"cannot read config file {path}")
    return config_from_parser(parser)


def loads_config(text: str) -> RunConfig:
    parser = configparser.ConfigParser(inline_comment_prefixes=("#", ";"))
    parser.read_string(text)
    return config_from_parser(parser)


def config_from_parser(parser: configparser.ConfigParser) -> RunConfig:
    v = parse_sections(parser)
    if v[("domain", "shape")] is not None and v[("domain", "bandwidth")] is None:
        raise ConfigError("[domain] shape given without bandwidth")
    try:
        problem = ProblemConfig(**{k: v[("problem", k)] for k in _dataclass_schema(ProblemConfig)})
        solver = SolverConfig(**{k: v[("optimizer", k)] for k in _dataclass_schema(SolverConfig)})
    except ValueError as exc:
        raise ConfigError(str(exc)) from exc
    objective, mode = v[("problem", "objective")], v[("problem", "mode")]
    if objective not in ("state", "deformation"):
        raise ConfigError(f"unknown objective {objective!r}")
    if mode not in ("stationary", "nonstationary"):
        raise ConfigError(f"unknown mode {mode!r}")
    cfg = RunConfig(problem=problem, solver=solver, objective=objective, mode=mode,
                    shape=v[("domain", "shape")], bandwidth=v[("domain", "bandwidth")],
                    alpha=v[("domain", "alpha")], order=v[("domain", "order")],
                    symbol=v[("domain", "symbol")], pad=v[("domain", "pad")], dtype=v[("domain", "dtype")],
                    **{k: v[("run", k)] for k in SCHEMA["run"]})
    if cfg.shape is not None:
        cfg.domain_for(cfg.shape)  # validate the domain eagerly
    return cfg


def effective_settings(cfg: RunConfig, domain: Domain) -> dict:
    """Every effective setting, defaults included (echoed into the report)."""
    out = {"domain.shape": " ".join(map(str, domain.shape)),
           "domain.bandwidth": " ".join(map(str, domain.bandwidth)),
           "domain.alpha": domain.alpha, "domain.order": domain.order, "domain.symbol": domain.symbol,
           "domain.pad": " ".join(map(str, domain.pad)), "domain.dtype": domain.dtype,
           "problem.objective": cfg.objective, "problem.mode": cfg.mode}
    out.update({f"problem.{k}": getattr(cfg.problem, k) for k in _dataclass_schema(ProblemConfig)})
    out.update({f"optimizer.{k}": getattr(cfg.solver, k) for k in _dataclass_schema(SolverConfig)})
    out["run.seed"] = cfg.seed
    return out
