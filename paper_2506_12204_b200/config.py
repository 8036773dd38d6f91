"""Scenario configuration as plain JSON-able dicts.

The reference's ``semsched.config`` API (``config.py:16-146``): the same
names (``ConfigError``, ``scenario_from_dict``, ``scenario_to_dict``,
``load_scenario``, ``apply_axis``), the same keys, defaults and error
behaviour, so a scenario file or a sweep axis means the same run on both
sides. The schema is declared once (``_SCHEMA``) and both directions are
driven from it.

Two reference behaviours kept on purpose: the workload seed is the
scenario's top-level ``seed`` (there is no ``workload.seed`` key), and
``apply_axis`` only wraps *unknown* axes in ``ConfigError`` -- a value that
does not parse as the key's type raises the plain ``ValueError`` of
``int()``/``float()``.
"""

from __future__ import annotations

import json
from typing import Any, Callable, Dict, Tuple

from .costs import profile_from_dict
from .engine import Policy, ScenarioConfig
from .predictors import PredictorConfig, Strategy
from .workload import WorkloadSpec


class ConfigError(ValueError):
    """Invalid or inconsistent scenario configuration."""


def _same(x):
    return x


# (section, key, parse, default, dump); section "" = top level
_Field = Tuple[str, str, Callable[[Any], Any], Any, Callable[[Any], Any]]
_SCHEMA: Tuple[_Field, ...] = (
    ("", "policy", Policy, "semantic", lambda v: v.value),
    ("", "profile", str, "a100_qwen7b", _same),
    ("", "batch_size", int, 16, _same),
    ("", "memory_capacity", int, 10**9, _same),
    ("", "seed", int, 0, _same),
    ("", "dependency_rule", bool, True, _same),
    ("", "decode_batch_cost", str, "max", _same),
    ("workload", "total_requests", int, 500, _same),
    ("workload", "gap_s", float, 0.2, _same),
    ("workload", "concurrent", int, 5, _same),
    ("workload", "concurrent_mode", str, "uniform", _same),
    ("workload", "levels", int, 5, _same),
    ("workload", "urgency_weights", _same, None, lambda v: list(v) if v else None),
    ("workload", "prompt_len_range", tuple, (16, 128), list),
    ("workload", "output_len_range", tuple, (1, 500), list),
    ("workload", "buckets", int, 5, _same),
    ("workload", "max_output_len", int, 500, _same),
    ("predictor", "latency_s", float, 0.0, _same),
    ("predictor", "batch_size", int, 64, _same),
    ("predictor", "strategy", Strategy, "immediate", lambda v: v.value),
    ("predictor", "urgency_error", float, 0.0, _same),
    ("predictor", "length_error", float, 0.0, _same),
)
_PROFILE_KEYS = ("alpha1", "alpha2", "gamma1", "gamma2", "beta_load", "beta_save")


def _owner(cfg: ScenarioConfig, section: str):
    return cfg if not section else getattr(cfg, section)


def scenario_from_dict(d: Dict[str, Any]) -> ScenarioConfig:
    """Build a ScenarioConfig from a scenario dict (missing keys take the
    defaults above); any malformed entry raises ``ConfigError``."""
    def section(name: str, src: Dict[str, Any]) -> Dict[str, Any]:
        return {key: parse(src.get(key, default)) for sec, key, parse, default, _ in _SCHEMA if sec == name}

    # evaluation order = the reference's, so the first error reported is the same
    try:
        wl_src, pred_src = dict(d.get("workload", {})), dict(d.get("predictor", {}))
        workload = WorkloadSpec(**section("workload", wl_src), seed=int(d.get("seed", 0)))
        predictor = PredictorConfig(**section("predictor", pred_src))
        override = None
        if "custom_profile" in d:
            override = profile_from_dict(d.get("profile", "custom"), d["custom_profile"])
        return ScenarioConfig(profile_override=override, workload=workload, predictor=predictor,
                              **section("", d))
    except (KeyError, TypeError, ValueError) as exc:
        raise ConfigError(str(exc)) from exc


def scenario_to_dict(cfg: ScenarioConfig) -> Dict[str, Any]:
    """The inverse of ``scenario_from_dict`` (the report's config echo)."""
    d: Dict[str, Any] = {"workload": {}, "predictor": {}}
    for section, key, _, _, dump in _SCHEMA:
        node = d if not section else d[section]
        node[key] = dump(getattr(_owner(cfg, section), key))
    if cfg.profile_override is not None:
        d["custom_profile"] = {k: getattr(cfg.profile_override, k) for k in _PROFILE_KEYS}
    return d


def load_scenario(path: str) -> ScenarioConfig:
    try:
        with open(path, "r", encoding="utf-8") as fh:
            d = json.load(fh)
    except (OSError, json.JSONDecodeError) as exc:
        raise ConfigError(f"cannot read scenario {path}: {exc}") from exc
    if not isinstance(d, dict):
        raise ConfigError("scenario file must hold a JSON object")
    return scenario_from_dict(d)


def _coerce(old: Any, value: str, axis: str) -> Any:
    # bool before int: bool is an int subclass
    if isinstance(old, bool):
        return value in ("1", "true", "True")
    if isinstance(old, int):
        return int(value)
    if isinstance(old, float):
        return float(value)
    if old is None or isinstance(old, str):
        return value
    raise ConfigError(f"axis {axis!r} is not a scalar")


def apply_axis(cfg: ScenarioConfig, axis: str, value: str) -> ScenarioConfig:
    """Copy of ``cfg`` with one dotted key (``seed``, ``workload.gap_s``,
    ``predictor.urgency_error``, ...) replaced by ``value`` parsed as the
    key's current type."""
    d = scenario_to_dict(cfg)
    *path, leaf = axis.split(".")
    node: Any = d
    for part in path:
        node = node.get(part) if isinstance(node, dict) else None
        if node is None:
            raise ConfigError(f"unknown axis {axis!r}")
    if not isinstance(node, dict) or leaf not in node:
        raise ConfigError(f"unknown axis {axis!r}")
    node[leaf] = _coerce(node[leaf], value, axis)
    return scenario_from_dict(d)
