"""The native async event loop (csrc/fs_async_engine.cpp) on CPU.

The loop never touches parameters, so it can be driven here with the CPU
oracle as the executor (test infrastructure only): the processed-event log
must replay the reference's golden digest (tests/golden/runs.json, made by
running the reference) and, on worlds without goldens (checkpointed
failures, horizons, k_min = 1), the oracle's own async engine
(oracle/fl_oracle.py OracleFederation.run_async, server.py:485-637).
"""

import math

import numpy as np
import pytest

from oracle import fl_oracle as O
from paper_2503_15448_b200 import async_loop
from paper_2503_15448_b200.config import ExperimentConfig
from paper_2503_15448_b200.experiment import build_world
from paper_2503_15448_b200.simnet import log_digest


class OracleExecutor:
    """Parameter work of the loop done by the oracle (numpy, serial)."""

    def __init__(self, world, w0):
        self.world = world
        self.sim = O.OracleFederation(world)
        self.versions = {0: np.asarray(w0, dtype=np.float64)}
        self.rows = {}
        self.reports = []
        self.aligned = []

    def aggregate(self, version, members):
        self.versions[version] = O.fedavg([self.rows[int(m)] for m in members])

    def report(self, info):
        self.reports.append(info)

    def train(self, ids, ci, cyc, ver):
        acc, rel = [], []
        rounds = self.world.rounds
        for i, c, k, v in zip(ids.tolist(), ci.tolist(), cyc.tolist(), ver.tolist()):
            wgp = self.versions[v - 1] if v > 0 else None
            o = self.sim.cycle(c, k, min(k, rounds - 1), self.versions[v], wgp)
            assert o["res"] is not None, "the loop deferred a cycle that does not train"
            self.rows[i] = o["res"]["params"]
            acc.append(o["accepted"])
            rel.append(math.nan if o["rel"] is None else o["rel"])
        return np.array(acc), np.array(rel)


def _native_run(world, w0, horizon=None):
    ex = OracleExecutor(world, w0)
    loop, y = async_loop.drive(world, ex, horizon if horizon is not None else world.horizon_s)
    block = loop.log_block()
    return ex, y, block


@pytest.mark.parametrize("name", ["async_weight", "async_delta_dyn", "async_fail_lost"])
def test_native_loop_replays_reference_digest(golden, name):
    run = golden("runs.json")[name]
    world, init = build_world(ExperimentConfig.from_dict(run["config"]))
    ex, y, block = _native_run(world, init.values)
    assert log_digest(block.records()) == run["digest"]
    assert len(block) == run["events"]
    want = golden("runs_wg.npz")[name]
    got = ex.versions[int(y.agg_count)]
    assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1.0)) < 1e-12
    assert [r["accepted"] for r in ex.reports] == [r["accepted"] for r in run["reports"]]
    assert [r["steps"] for r in ex.reports] == [r["sgd_steps"] for r in run["reports"]]


def _cfg(**over):
    cfg = {"num_clients": 6, "rounds": 3, "epochs": 1, "mode": "async_filtered", "selection_mode": "weight_sign",
           "dataset": {"n": 900, "d": 6}, "model": {"hidden_dims": [8], "dropout_rate": 0.2}, "seed": 3,
           "batch": {"policy": "fixed", "size": 32},
           "profiles": {"speed": {"distribution": "loguniform", "low": 20.0, "high": 200.0},
                        "up_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5},
                        "down_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5}}}
    for k, v in over.items():
        if isinstance(v, dict) and isinstance(cfg.get(k), dict):
            cfg[k] = {**cfg[k], **v}
        else:
            cfg[k] = v
    return cfg


@pytest.mark.parametrize("over", [
    {},
    {"selection_mode": "delta_sign", "aggregation": {"k_min": 1}},
    {"dropout_rate": 0.3, "checkpoint": {"enabled": True, "total_time_s": 20.0, "recovery_s": 0.7}},
    {"dropout_rate": 0.3},
    {"async_run": {"horizon_s": 4.0, "cycle_cap": 50}},
    {"async_run": {"horizon_s": None, "cycle_cap": 1}, "rounds": 4},
    {"aggregation": {"k_min": 3, "timeout_s": 0.2}},
    {"theta": 0.99, "async_run": {"horizon_s": None, "cycle_cap": 1}},
])
def test_native_loop_matches_oracle_engine(over):
    try:
        world, init = build_world(ExperimentConfig.from_dict(_cfg(**over)))
    except (KeyError, ValueError) as e:  # config key not supported by this builder
        pytest.skip(f"config not expressible: {e}")
    sim = O.OracleFederation(world)
    wg = sim.run(init.values)
    ex, y, block = _native_run(world, init.values)
    recs = block.records()
    assert log_digest(recs) == sim.digest()
    assert len(recs) == len(sim.clock.log)
    got = ex.versions[int(y.agg_count)] if y.agg_count else init.values
    assert np.array_equal(got, wg)
    assert len(ex.reports) == len(sim.reports)
    for a, b in zip(ex.reports, sim.reports):
        assert (a["accepted"], a["rejected"], a["failures"], a["steps"]) == \
               (b["accepted"], b["rejected"], b["failures"], b["sgd_steps"])
        assert a["aggregations"] == b["aggregations"]


def test_native_loop_rejects_bad_provide():
    world, init = build_world(ExperimentConfig.from_dict(_cfg()))
    loop = async_loop.AsyncLoop(world, None)
    assert loop.run() == async_loop.NEED_EVAL
    ids, _, _, _ = loop.pending()
    with pytest.raises(ValueError):
        loop.provide(np.ones(len(ids) + 1, dtype=bool), np.zeros(len(ids) + 1))
    loop.close()
