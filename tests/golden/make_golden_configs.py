"""Golden fixtures at the BASELINE.json configurations, recorded from the
REFERENCE package itself (oracle/_ref/pkg with its compiled Cython backend,
built by oracle/build_ref.sh from /root/reference).

Configs (the same dicts as bench.py):
  c1_sync      configs[0]: UNSW-shaped d=42, MLP 256-128-64, 10 clients,
               5 rounds, sync_baseline, fixed b=64
  c2_async     configs[1]: 100 clients, async_filtered, dynamic batch,
               delta_sign theta=0.65, 2 windows (of 5; ~2 min on one core)
  c3_sync      configs[2]: ROAD-shaped d=64, 256 clients, sync_filtered,
               delta_sign, b=64, 2 rounds
  c4_sync      configs[3]: 1024 UNSW-shaped clients, sync_filtered, dynamic
               batch, delta_sign, 5 rounds -- plus the global model after
               EVERY round (the teacher-forcing sequence of the bf16 parity
               protocol) and every round's aligned counts

Recorded per config: replay digest, event count, per-round aligned counts
of every scored client (from the train_done records: aligned =
relevance * M, exact), per-round reports (accuracy/AUC/...), the final
global model (and for c4 all round models) as float64.

Sync rounds fan the clients out over forked processes
(oracle/ref_pool.ForkPoolExecutor in place of the reference's thread pool):
each client cycle is a pure function, so the result equals the serial run's
(the c1 digest is also reproduced serially below as a check).

Usage:  oracle/build_ref.sh && python tests/golden/make_golden_configs.py
Writes tests/golden/configs.json and tests/golden/configs_wg.npz.
"""

from __future__ import annotations

import copy
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

PROF = {"speed": {"distribution": "loguniform", "low": 20.0, "high": 200.0},
        "capacity": {"distribution": "loguniform", "low": 0.25, "high": 4.0},
        "up_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5},
        "down_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5}}
UNSW = {"kind": "synthetic", "n": 219176, "d": 42, "anomaly_frac": 0.3, "separation": 4.0, "test_frac": 0.2}
ROAD = {"kind": "synthetic", "d": 64, "samples_per_client": 256, "anomaly_frac": 0.1, "separation": 2.0,
        "test_frac": 0.2}
MLP = {"hidden_dims": [256, 128, 64], "dropout_rate": 0.3}
DYN = {"policy": "dynamic", "b_ref": 64, "b_min": 64, "b_max": 1024}
BASE = {"epochs": 5, "lr": 0.05, "lr_decay": 0.9, "seed": 1, "profiles": PROF, "model": MLP}

CONFIGS = {
    "c1_sync": dict(BASE, num_clients=10, rounds=5, mode="sync_baseline", dataset=UNSW,
                    batch={"policy": "fixed", "size": 64}),
    "c2_async": dict(BASE, num_clients=100, rounds=2, mode="async_filtered", dataset=UNSW, batch=DYN,
                     selection_mode="delta_sign", theta=0.65),
    "c3_sync": dict(BASE, num_clients=256, rounds=2, mode="sync_filtered", dataset=ROAD,
                    batch={"policy": "fixed", "size": 64}, selection_mode="delta_sign", theta=0.65),
    "c4_sync": dict(BASE, num_clients=1024, rounds=5, mode="sync_filtered", dataset=UNSW, batch=DYN,
                    selection_mode="delta_sign", theta=0.65),
}


def aligned_by_round(log, M):
    out = {}
    for rec in log:
        if rec["kind"] == "train_done" and rec.get("relevance") is not None:
            out.setdefault(str(rec["round"]), []).append((rec["client_id"], int(round(rec["relevance"] * M))))
    return {r: [a for _, a in sorted(v)] for r, v in out.items()}, \
           {r: [c for c, _ in sorted(v)] for r, v in out.items()}


def run_config(name, cfg, workers):
    from fedsim.config import ExperimentConfig
    from fedsim.experiment import build_world
    from fedsim.server import FederationEngine, GlobalState

    world, initial = build_world(ExperimentConfig.from_dict(cfg), workers=workers)
    M = world.spec.param_count
    eng = FederationEngine(world)
    t0 = time.perf_counter()
    models = [initial.values.copy()]
    if world.mode == "async_filtered":
        state = eng.run(initial)
    else:
        state = GlobalState(round=0, w_g=initial)
        for _ in range(world.rounds):
            state = eng.run_sync_round(state)
            models.append(state.w_g.values.copy())
        eng.timeline.schedule(eng.timeline.now_s, "run_end", reason="rounds_done")
        eng.timeline.run(eng._record)
    wall = time.perf_counter() - t0
    aligned, clients = aligned_by_round(list(eng.timeline.log), M)
    rec = {"config": cfg, "digest": eng.timeline.digest(), "events": len(eng.timeline.log), "M": M,
           "aligned": aligned, "aligned_clients": clients,
           "reports": [r.to_record() for r in eng.reports], "wall_s": wall, "workers": workers}
    print(f"{name}: digest {rec['digest']} events {rec['events']} wall {wall:.1f}s", flush=True)
    return rec, state.w_g.values.copy(), np.stack(models)


def main() -> None:
    from oracle.ref_pool import patch_server_pool, use_reference

    use_reference("compiled")
    import fedsim.server

    patch_server_pool(fedsim.server)
    workers = os.cpu_count() or 1
    recs, arrays = {}, {}
    for name, cfg in CONFIGS.items():
        rec, wg, models = run_config(name, copy.deepcopy(cfg), workers)
        recs[name] = rec
        arrays[f"{name}_wg"] = wg
        if name == "c4_sync":
            arrays["c4_sync_models"] = models  # w_g after rounds 0..5 (index 0 = initial)
    # the fork pool reproduces the serial run (c1: 10 clients, serial ~80 s)
    serial, _, _ = run_config("c1_sync(serial)", copy.deepcopy(CONFIGS["c1_sync"]), 1)
    assert serial["digest"] == recs["c1_sync"]["digest"], "fork pool changed the reference's result"
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump(recs, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "configs_wg.npz"), **arrays)


if __name__ == "__main__":
    main()
