"""Experiment configuration: the reference schema, deep-merged over defaults.

Same keys, defaults and merge rules as pkg/src/fedsim/config.py:16-176 so a
config file drives both this framework and the reference identically
(unknown keys rejected with their field path; profile distributions and
label mappings replaced wholesale). Validation covers the fields the round
loop consumes.
"""

from __future__ import annotations

import copy
import json
from dataclasses import dataclass

DEFAULTS: dict = {
    "dataset": {
        "kind": "synthetic", "n": 20000, "d": 20, "anomaly_frac": 0.3, "separation": 4.0,
        "samples_per_client": None, "path": None, "label_column": "label",
        "categorical_columns": [], "label_mapping": None, "test_frac": 0.2,
    },
    "partition": {"alpha": 0.5, "fraction": 1.0},
    "num_clients": 10,
    "rounds": 6,
    "epochs": 5,
    "model": {"hidden_dims": [256, 128, 64], "dropout_rate": 0.3},
    "batch": {"policy": "fixed", "size": 64, "b_ref": 64, "b_min": 64, "b_max": 1024},
    "mode": "sync_filtered",
    "theta": 0.65,
    "selection_mode": "weight_sign",
    "profiles": {
        "speed": {"distribution": "constant", "value": 50.0},
        "capacity": {"distribution": "constant", "value": 1.0},
        "up_latency": {"distribution": "constant", "value": 1.0},
        "down_latency": {"distribution": "constant", "value": 1.0},
    },
    "dropout_rate": 0.0,
    "weibull": {"lambda_s": 300.0, "k": 1.5},
    "checkpoint": {"enabled": False, "total_time_s": 600.0, "recovery_s": 5.0, "grid_s": None},
    "aggregation": {"k_min": 2, "timeout_s": 5.0, "cost_per_update_s": 0.05},
    "step_overhead_s": 0.0,
    "async_run": {"horizon_s": None, "cycle_cap": 50},
    "lr": 0.05,
    "lr_decay": 0.9,
    "seed": 1,
    # framework extensions (north-star opt-ins; none is on the reference's
    # parity path and none exists in the reference schema: a config that
    # leaves them at these defaults serialises without this section)
    "extensions": {
        "top_k": None,             # at most k accepted clients per sync round
        "staleness_alpha": None,   # async FedAvg weights (1 + staleness) ** -alpha
        "optimizer": "sgd",        # "sgd" | "adam" (local optimizer)
        "adam": {"beta1": 0.9, "beta2": 0.999, "eps": 1e-8},
    },
}

MODES = ("sync_baseline", "sync_filtered", "async_filtered")
ATOMIC_PATHS = {
    "profiles.speed", "profiles.capacity", "profiles.up_latency", "profiles.down_latency",
    "dataset.label_mapping",
}


class ConfigError(ValueError):
    """Invalid configuration, with a field-path message."""


def _merge(defaults: dict, override, path: str = "") -> dict:
    if not isinstance(override, dict):
        raise ConfigError(f"{path or 'config'}: expected an object, got {type(override).__name__}")
    out = copy.deepcopy(defaults)
    for key, value in override.items():
        here = f"{path}.{key}" if path else key
        if key not in defaults:
            raise ConfigError(f"{here}: unknown key")
        nested = isinstance(defaults[key], dict) and defaults[key] and here not in ATOMIC_PATHS
        out[key] = _merge(defaults[key], value, here) if nested else copy.deepcopy(value)
    return out


def _need(cond: bool, path: str, msg: str) -> None:
    if not cond:
        raise ConfigError(f"{path}: {msg}")


def _pow2(x) -> bool:
    return isinstance(x, int) and x >= 1 and (x & (x - 1)) == 0


def validate(cfg: dict) -> None:
    ds = cfg["dataset"]
    _need(ds["kind"] == "synthetic", "dataset.kind", "only synthetic datasets feed this framework")
    _need(0 < ds["test_frac"] < 1, "dataset.test_frac", "must be in (0,1)")
    _need(int(ds["d"]) >= 1, "dataset.d", "must be >= 1")
    _need(0 < ds["anomaly_frac"] < 1, "dataset.anomaly_frac", "must be in (0,1)")
    _need(cfg["partition"]["alpha"] > 0, "partition.alpha", "must be > 0")
    _need(0 < cfg["partition"]["fraction"] <= 1, "partition.fraction", "must be in (0,1]")
    _need(int(cfg["num_clients"]) >= 1, "num_clients", "must be >= 1")
    _need(int(cfg["rounds"]) >= 0, "rounds", "must be >= 0")
    _need(int(cfg["epochs"]) >= 0, "epochs", "must be >= 0")
    hd = cfg["model"]["hidden_dims"]
    _need(isinstance(hd, list) and hd and all(isinstance(h, int) and h >= 1 for h in hd),
          "model.hidden_dims", "must be a non-empty list of positive integers")
    _need(len(hd) + 1 <= 8, "model.hidden_dims", "at most 7 hidden layers")
    _need(0 <= cfg["model"]["dropout_rate"] < 1, "model.dropout_rate", "must be in [0,1)")
    b = cfg["batch"]
    _need(b["policy"] in ("fixed", "dynamic"), "batch.policy", "must be 'fixed' or 'dynamic'")
    for key in ("size", "b_ref", "b_min", "b_max"):
        _need(_pow2(b[key]), f"batch.{key}", "must be a positive power of two")
    _need(b["b_min"] <= b["b_ref"] <= b["b_max"], "batch.b_ref", "needs b_min <= b_ref <= b_max")
    _need(cfg["mode"] in MODES, "mode", f"must be one of {MODES}")
    _need(cfg["selection_mode"] in ("weight_sign", "delta_sign", "delta_cosine"), "selection_mode",
          "must be 'weight_sign', 'delta_sign' or 'delta_cosine'")
    lo = -1 if cfg["selection_mode"] == "delta_cosine" else 0
    _need(lo <= cfg["theta"] <= 1, "theta", f"must be in [{lo},1]")
    ext = cfg["extensions"]
    _need(ext["top_k"] is None or (isinstance(ext["top_k"], int) and ext["top_k"] >= 1), "extensions.top_k",
          "must be a positive int or null")
    _need(ext["staleness_alpha"] is None or ext["staleness_alpha"] >= 0, "extensions.staleness_alpha",
          "must be >= 0 or null")
    _need(ext["optimizer"] in ("sgd", "adam"), "extensions.optimizer", "must be 'sgd' or 'adam'")
    ad = ext["adam"]
    _need(0 <= ad["beta1"] < 1 and 0 <= ad["beta2"] < 1 and ad["eps"] > 0, "extensions.adam",
          "needs 0 <= beta1, beta2 < 1 and eps > 0")
    _need(0 <= cfg["dropout_rate"] <= 1, "dropout_rate", "must be in [0,1]")
    agg = cfg["aggregation"]
    _need(int(agg["k_min"]) >= 1, "aggregation.k_min", "must be >= 1")
    _need(agg["timeout_s"] > 0, "aggregation.timeout_s", "must be > 0")
    _need(agg["cost_per_update_s"] >= 0, "aggregation.cost_per_update_s", "must be >= 0")
    _need(int(cfg["async_run"]["cycle_cap"]) >= 1, "async_run.cycle_cap", "must be >= 1")
    _need(cfg["lr"] > 0, "lr", "must be > 0")
    _need(0 < cfg["lr_decay"] <= 1, "lr_decay", "must be in (0,1]")
    _need(isinstance(cfg["seed"], int) and cfg["seed"] >= 0, "seed", "must be a non-negative int")


@dataclass(frozen=True)
class ExperimentConfig:
    raw: dict

    @staticmethod
    def from_dict(d: dict) -> "ExperimentConfig":
        cfg = _merge(DEFAULTS, d)
        validate(cfg)
        return ExperimentConfig(cfg)

    @staticmethod
    def from_file(path: str) -> "ExperimentConfig":
        with open(path, encoding="utf-8") as f:
            return ExperimentConfig.from_dict(json.load(f))

    def to_dict(self) -> dict:
        d = copy.deepcopy(self.raw)
        if d.get("extensions") == DEFAULTS["extensions"]:
            del d["extensions"]  # the reference schema has no such section
        return d

    def canonical_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True, indent=2) + "\n"

    def with_overrides(self, **top) -> "ExperimentConfig":
        d = self.to_dict()
        for k, v in top.items():
            if isinstance(v, dict) and isinstance(d.get(k), dict):
                d[k].update(v)
            else:
                d[k] = v
        return ExperimentConfig.from_dict(d)

    def __getitem__(self, key):
        return self.raw[key]

    @property
    def seed(self) -> int:
        return self.raw["seed"]

    @property
    def mode(self) -> str:
        return self.raw["mode"]

    @property
    def num_clients(self) -> int:
        return self.raw["num_clients"]
