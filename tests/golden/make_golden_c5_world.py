"""Digest of the BASELINE configs[4] (C5) world as the REFERENCE package builds
it: 8192 UNSW-shaped clients, Dirichlet alpha = 5.0 (alpha = 0.5 fails to
partition at 8192 clients), WIDE MLP 42-1024x4-1, b = 64,
async_filtered, delta_sign. Only the world is recorded: the reference cannot
train it (its update stack needs ~209 GB).

Usage:  oracle/build_ref.sh && python tests/golden/make_golden_c5_world.py
Writes tests/golden/c5_world.json.
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

C5 = {"num_clients": 8192, "rounds": 5, "epochs": 5, "mode": "async_filtered", "selection_mode": "delta_sign",
      "theta": 0.65, "seed": 1, "lr": 0.05, "lr_decay": 0.9,
      "dataset": {"kind": "synthetic", "n": 219176, "d": 42, "anomaly_frac": 0.3, "separation": 4.0,
                  "test_frac": 0.2},
      "partition": {"alpha": 5.0},
      "model": {"hidden_dims": [1024, 1024, 1024, 1024], "dropout_rate": 0.3},
      "batch": {"policy": "fixed", "size": 64},
      "profiles": {"speed": {"distribution": "loguniform", "low": 20.0, "high": 200.0},
                   "capacity": {"distribution": "loguniform", "low": 0.25, "high": 4.0},
                   "up_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5},
                   "down_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5}}}


def main() -> None:
    from oracle.ref_pool import use_reference

    use_reference("compiled")
    from fedsim.config import ExperimentConfig
    from fedsim.experiment import build_world

    from tests.golden.make_golden import world_digest

    t0 = time.perf_counter()
    world, initial = build_world(ExperimentConfig.from_dict(C5))
    n = [wc.features.shape[0] for wc in world.clients]
    rec = {"config": C5, "digest": world_digest(world, initial), "param_count": world.spec.param_count,
           "rows_min": min(n), "rows_max": max(n), "rows_total": sum(n), "build_s": time.perf_counter() - t0}
    print(json.dumps(rec)[-300:])
    with open(os.path.join(HERE, "c5_world.json"), "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
