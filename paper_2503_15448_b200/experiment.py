"""Experiment wiring: config -> world -> engine (one-time host work).

``build_world`` follows pkg/src/fedsim/experiment.py:74-202 stream for
stream (dataset, stratified split, Dirichlet partition, per-client
profiles, capacity-driven batch sizes, checkpoint interval, geometry,
failure schedule, initial parameters), so a config yields the same world
as in the reference; tests/golden pins the digests. ``run_experiment``
drives the engine, returns the replay digest, summary and final parameters
and writes the reference's run-directory artifacts; ``replay_run`` re-runs
a directory and compares digests.
"""

from __future__ import annotations

import hashlib
import json
import os
import time
from dataclasses import dataclass

import numpy as np

from . import __version__
from .backends import backend_name
from .client import ClientProfile, assign_batch_size
from .config import ExperimentConfig
from .data import partition_dirichlet, stratified_split, synth_anomaly
from .fault import (CheckpointPolicy, WeibullModel, failure_offsets, inject_dropout, optimal_interval,
                    write_checkpoint_file)
from .model import ModelSpec, ParamVector, init_params
from .rng import derive_rng, derive_seed
from .selection import SelectionPolicy
from .server import FederationEngine, World, WorldClient, finalize_client_geometry
from .metrics import summarize_reports, write_reports
from .simnet import DistSpec, write_event_log


def params_digest(params: ParamVector) -> str:
    return hashlib.blake2b(params.values.tobytes(), digest_size=8).hexdigest()


def load_dataset(config: ExperimentConfig):
    ds = config["dataset"]
    n = ds["n"]
    if ds["samples_per_client"] is not None:
        n = int(round(ds["samples_per_client"] * config.num_clients / (1.0 - ds["test_frac"])))
    return synth_anomaly(n=n, d=ds["d"], anomaly_frac=ds["anomaly_frac"], separation=ds["separation"],
                         seed=derive_seed(config.seed, "data"))


def build_world(config: ExperimentConfig, workers: int = 1, precision: str = "fp64") -> tuple[World, ParamVector]:
    cfg = config.raw
    seed = config.seed
    ds = load_dataset(config)
    train_idx, test_idx = stratified_split(ds, cfg["dataset"]["test_frac"], seed)
    part = partition_dirichlet(ds, config.num_clients, cfg["partition"]["alpha"], seed,
                               indices=train_idx, fraction=cfg["partition"]["fraction"])
    dists = {k: DistSpec.from_config(cfg["profiles"][k]) for k in ("speed", "capacity", "up_latency", "down_latency")}
    weibull = WeibullModel(cfg["weibull"]["lambda_s"], cfg["weibull"]["k"])
    profiles = []
    for i in range(config.num_clients):
        rng = derive_rng(seed, "profile", i)
        speed = dists["speed"].sample(rng)
        capacity = dists["capacity"].sample(rng)
        up = dists["up_latency"].sample(rng)
        down = dists["down_latency"].sample(rng)
        profiles.append(ClientProfile(id=i, speed=speed, capacity=capacity, up_latency_s=up,
                                      down_latency_s=down, dropout_rate=cfg["dropout_rate"], weibull=weibull))
    bc = cfg["batch"]
    if bc["policy"] == "dynamic":
        cap_ref = float(np.mean([p.capacity for p in profiles]))
        sizes = [assign_batch_size(p, bc["b_ref"], cap_ref, bc["b_min"], bc["b_max"]) for p in profiles]
    else:
        sizes = [bc["size"]] * config.num_clients
    ck = cfg["checkpoint"]
    interval = None
    if ck["enabled"]:
        grid = ck["grid_s"] if ck["grid_s"] is not None else ck["total_time_s"] / 1000.0
        interval = optimal_interval(CheckpointPolicy(t_c_s=grid, total_time_s=ck["total_time_s"],
                                                     recovery_s=ck["recovery_s"]), weibull, grid)
    clients = []
    for p, b in zip(profiles, sizes):
        idx = part.assignments[p.id]
        wc = WorldClient(profile=p, features=ds.features[idx], labels=ds.labels[idx], batch_size=b)
        finalize_client_geometry(wc, cfg["epochs"], cfg["step_overhead_s"], interval)
        clients.append(wc)
    theta = 0.0 if config.mode == "sync_baseline" else cfg["theta"]
    cycles = cfg["rounds"] * cfg["async_run"]["cycle_cap"]
    world = World(
        spec=ModelSpec(input_dim=ds.dim, hidden_dims=tuple(cfg["model"]["hidden_dims"]),
                       dropout_rate=cfg["model"]["dropout_rate"]),
        clients=clients, test_features=ds.features[test_idx], test_labels=ds.labels[test_idx],
        policy=SelectionPolicy(theta=theta, mode=cfg["selection_mode"], top_k=cfg["extensions"]["top_k"]),
        mode=config.mode,
        epochs=cfg["epochs"], rounds=cfg["rounds"], base_lr=cfg["lr"], lr_decay=cfg["lr_decay"],
        agg_cost_per_update_s=cfg["aggregation"]["cost_per_update_s"], k_min=cfg["aggregation"]["k_min"],
        buffer_timeout_s=cfg["aggregation"]["timeout_s"], master_seed=seed, dropout_rate=cfg["dropout_rate"],
        fail_matrix=inject_dropout(config.num_clients, cycles, cfg["dropout_rate"], seed),
        fail_offsets=failure_offsets(config.num_clients, cycles, seed),
        checkpointing=ck["enabled"], recovery_s=ck["recovery_s"], step_overhead_s=cfg["step_overhead_s"],
        workers=workers, horizon_s=cfg["async_run"]["horizon_s"], cycle_cap=cfg["async_run"]["cycle_cap"],
        precision=precision,
        staleness_alpha=cfg["extensions"]["staleness_alpha"], optimizer=cfg["extensions"]["optimizer"],
        adam=(cfg["extensions"]["adam"]["beta1"], cfg["extensions"]["adam"]["beta2"], cfg["extensions"]["adam"]["eps"]),
    )
    return world, init_params(world.spec, derive_seed(seed, "model-init"))


@dataclass
class RunResult:
    config: ExperimentConfig
    world: World
    engine: FederationEngine
    reports: list
    final_params: ParamVector
    digest: str
    summary: dict
    wall_clock_s: float

    @property
    def final_accuracy(self) -> float:
        return self.reports[-1].accuracy if self.reports else float("nan")

    @property
    def final_auc(self) -> float:
        return self.reports[-1].auc if self.reports else float("nan")


def run_experiment(config: ExperimentConfig, out_dir: str | None = None, workers: int = 1, *,
                   world_and_initial=None, precision: str = "fp64") -> RunResult:
    """Build a world, run it, and (with ``out_dir``) write the run directory
    (reference experiment.py:206-272): ``config.json``, ``events.jsonl``,
    ``rounds.jsonl``, ``summary.csv``, ``run_meta.json`` and the final global
    checkpoint (``checkpoints/`` + MANIFEST.json).

    ``workers`` is accepted for API compatibility (clients are batched on the
    device; results do not depend on it). Framework extensions are
    keyword-only: ``world_and_initial`` reuses a prebuilt ``build_world``
    result, ``precision`` selects the fp64 parity or bf16 trainer."""
    t0 = time.perf_counter()
    world, initial = (world_and_initial if world_and_initial is not None
                      else build_world(config, workers=workers, precision=precision))
    engine = FederationEngine(world)
    state = engine.run(initial)
    wall = time.perf_counter() - t0
    digest = engine.timeline.digest()
    extra = {"seed": config.seed, "mode": config.mode, "theta": world.policy.theta}
    result = RunResult(config, world, engine, engine.reports, state.w_g, digest, {}, wall)
    if out_dir is None:
        result.summary = summarize_reports(engine.reports, extra)
        return result
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "config.json"), "w", encoding="utf-8") as f:
        f.write(config.canonical_json())
    write_event_log(list(engine.timeline.log), os.path.join(out_dir, "events.jsonl"))
    result.summary = write_reports(engine.reports, out_dir, extra)
    meta = {"digest": digest, "params_digest": params_digest(state.w_g), "backend": backend_name(),
            "version": __version__, "events": len(engine.timeline.log), "wall_clock_s": wall,
            "workers": workers, "precision": world.precision}
    with open(os.path.join(out_dir, "run_meta.json"), "w", encoding="utf-8") as f:
        json.dump(meta, f, indent=2, sort_keys=True)
    if engine.global_checkpoints:
        write_checkpoint_file(engine.global_checkpoints[-1], os.path.join(out_dir, "checkpoints"))
    return result


def replay_run(run_dir: str, workers: int = 1) -> tuple[bool, dict]:
    """Re-run a run directory's config and compare the replay and parameter
    digests with the recorded ones (reference experiment.py:275-296)."""
    config = ExperimentConfig.from_file(os.path.join(run_dir, "config.json"))
    with open(os.path.join(run_dir, "run_meta.json"), encoding="utf-8") as f:
        meta = json.load(f)
    result = run_experiment(config, None, workers, precision=meta.get("precision", "fp64"))
    report = {"recorded_digest": meta["digest"], "replayed_digest": result.digest,
              "recorded_params_digest": meta.get("params_digest"),
              "replayed_params_digest": params_digest(result.final_params),
              "recorded_backend": meta.get("backend"), "active_backend": backend_name()}
    ok = (report["recorded_digest"] == report["replayed_digest"]
          and report["recorded_params_digest"] == report["replayed_params_digest"])
    return ok, report
