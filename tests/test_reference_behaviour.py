"""Reference behaviours (pkg/tests/test_server.py, test_client.py,
test_selection.py, test_simnet.py) re-checked against this framework's API.

Host-only behaviours run everywhere; engine behaviours need the GPU (the
framework has no CPU execution path).
"""

import math

import numpy as np
import pytest

from tests.conftest import cuda_ok



# ------------------------------------------------------------------ host-only
def _profile(cid=0, speed=50.0, capacity=1.0):
    from paper_2503_15448_b200.client import ClientProfile

    return ClientProfile(id=cid, speed=speed, up_latency_s=1.0, down_latency_s=1.0, capacity=capacity)


def test_batch_size_assignment_cases():
    # reference tests/test_client.py:35-63 (paper cases 512 / 64, monotone, validation)
    from paper_2503_15448_b200.client import assign_batch_size

    assert assign_batch_size(_profile(capacity=2.0), 64, 2.0, 64, 512) == 64
    assert assign_batch_size(_profile(capacity=8.0), 64, 1.0, 64, 512) == 512
    assert assign_batch_size(_profile(capacity=1e-9), 256, 1.0, 64, 512) == 64
    sizes = [assign_batch_size(_profile(capacity=c), 128, 1.0, 32, 1024) for c in np.linspace(0.05, 16.0, 60)]
    assert all(b >= a for a, b in zip(sizes, sizes[1:]))
    with pytest.raises(ValueError):
        assign_batch_size(_profile(), 48, 1.0, 32, 512)
    with pytest.raises(ValueError):
        assign_batch_size(_profile(), 64, 1.0, 128, 512)


def test_profile_and_spec_validation():
    from paper_2503_15448_b200.client import ClientProfile
    from paper_2503_15448_b200.model import ModelSpec
    from paper_2503_15448_b200.selection import SelectionPolicy

    with pytest.raises(ValueError):
        ClientProfile(id=0, speed=0.0, up_latency_s=0, down_latency_s=0, capacity=1)
    with pytest.raises(ValueError):
        ClientProfile(id=0, speed=1.0, up_latency_s=-1, down_latency_s=0, capacity=1)
    with pytest.raises(ValueError):
        ModelSpec(input_dim=0, hidden_dims=(4,))
    with pytest.raises(ValueError):
        ModelSpec(input_dim=3, hidden_dims=())
    with pytest.raises(ValueError):
        ModelSpec(input_dim=3, hidden_dims=(4,), dropout_rate=1.0)
    with pytest.raises(ValueError):
        SelectionPolicy(theta=1.5)
    with pytest.raises(ValueError):
        SelectionPolicy(mode="cosine")
    assert ModelSpec(input_dim=3, hidden_dims=(4,)).param_count == 4 * 4 + 5 * 1  # reference test_model.py:73-76


def test_time_law_batch_count_lr_schedule():
    from paper_2503_15448_b200.client import batch_count, train_time_law
    from paper_2503_15448_b200.model import lr_schedule

    assert batch_count(100, 16) == 7 and batch_count(64, 64) == 1
    assert train_time_law(5, 100, 50.0) == 10.0
    assert lr_schedule(2, 0.1, 0.5) == pytest.approx(0.025)  # reference test_model.py:312-319
    with pytest.raises(ValueError):
        lr_schedule(-1, 0.1, 0.5)
    with pytest.raises(ValueError):
        lr_schedule(0, 0.1, 0.0)


def test_timeline_ordering_stop_and_horizon():
    # reference tests/test_simnet.py
    from paper_2503_15448_b200.simnet import Timeline, log_digest

    tl = Timeline()
    for t, k in ((2.0, "upload_arrive"), (1.0, "train_done"), (1.0, "aggregate")):
        tl.schedule(t, k)
    seen = []
    tl.run(lambda ev: seen.append((ev.t_s, ev.kind)) or {"kind": ev.kind, "t_s": ev.t_s})
    assert seen == [(1.0, "train_done"), (1.0, "aggregate"), (2.0, "upload_arrive")]
    with pytest.raises(ValueError):
        tl.schedule(0.5, "aggregate")
    with pytest.raises(ValueError):
        tl.schedule(3.0, "not_a_kind")
    tl2 = Timeline()
    tl2.schedule(1.0, "checkpoint")
    tl2.schedule(5.0, "checkpoint")
    assert tl2.run(lambda ev: None, horizon_s=3.0) == 1 and tl2.now_s == 3.0
    tl3 = Timeline()
    tl3.schedule(1.0, "run_end")
    tl3.schedule(2.0, "checkpoint")
    tl3.run(lambda ev: tl3.stop() or {"k": 1})
    assert tl3.stopped and len(tl3.log) == 1
    a = log_digest([{"a": 1}, {"b": 2}])
    assert a != log_digest([{"b": 2}, {"a": 1}])


def test_distspec_draws_match_numpy():
    from paper_2503_15448_b200.simnet import DistSpec

    rng_a, rng_b = np.random.default_rng(3), np.random.default_rng(3)
    d = DistSpec.from_config({"distribution": "loguniform", "low": 20.0, "high": 200.0})
    assert d.sample(rng_a) == float(math.exp(rng_b.uniform(math.log(20.0), math.log(200.0))))
    with pytest.raises(ValueError):
        DistSpec.from_config({"distribution": "loguniform", "low": 0.0, "high": 1.0})
    with pytest.raises(ValueError):
        DistSpec.from_config({"distribution": "gamma"})


def test_config_merge_rejects_unknown_keys():
    from paper_2503_15448_b200.config import ConfigError, ExperimentConfig

    with pytest.raises(ConfigError):
        ExperimentConfig.from_dict({"dataset": {"nope": 1}})
    with pytest.raises(ConfigError):
        ExperimentConfig.from_dict({"batch": {"size": 48}})
    cfg = ExperimentConfig.from_dict({"profiles": {"speed": {"distribution": "constant", "value": 3.0}}})
    assert cfg["profiles"]["speed"] == {"distribution": "constant", "value": 3.0}
    assert cfg.with_overrides(rounds=2)["rounds"] == 2


# ------------------------------------------------------------------ engines (GPU)
def make_world(speeds, mode="sync_filtered", theta=0.0, rounds=1, epochs=1, up=0.0, down=0.0, a_s=0.0,
               n_rows=10, k_min=1, dropout=0.0, seed=99, cycle_cap=50, timeout_s=5.0):
    """Hand-built world with per-client speeds (after reference tests/test_server.py:78-134)."""
    from paper_2503_15448_b200.client import ClientProfile
    from paper_2503_15448_b200.fault import failure_offsets, inject_dropout
    from paper_2503_15448_b200.model import ModelSpec, init_params
    from paper_2503_15448_b200.selection import SelectionPolicy
    from paper_2503_15448_b200.server import World, WorldClient, finalize_client_geometry

    spec = ModelSpec(input_dim=3, hidden_dims=(4,), dropout_rate=0.0)
    rng = np.random.default_rng(5)
    clients = []
    for i, speed in enumerate(speeds):
        wc = WorldClient(profile=ClientProfile(id=i, speed=speed, up_latency_s=up, down_latency_s=down, capacity=1.0),
                         features=rng.normal(size=(n_rows, 3)), labels=rng.integers(0, 2, n_rows).astype(np.int8),
                         batch_size=n_rows)
        finalize_client_geometry(wc, epochs, 0.0, None)
        clients.append(wc)
    cycles = rounds * cycle_cap
    world = World(spec=spec, clients=clients, test_features=rng.normal(size=(20, 3)),
                  test_labels=rng.integers(0, 2, 20).astype(np.int8), policy=SelectionPolicy(theta=theta),
                  mode=mode, epochs=epochs, rounds=rounds, base_lr=0.1, lr_decay=1.0, agg_cost_per_update_s=a_s,
                  k_min=k_min, buffer_timeout_s=timeout_s, master_seed=seed, dropout_rate=dropout,
                  fail_matrix=inject_dropout(len(speeds), cycles, dropout, seed),
                  fail_offsets=failure_offsets(len(speeds), cycles, seed), cycle_cap=cycle_cap)
    return world, init_params(spec, 1)


def _run(world, w0):
    from paper_2503_15448_b200.server import FederationEngine

    eng = FederationEngine(world)
    state = eng.run(w0)
    return eng, state


def _kind(eng, k):
    return [r for r in eng.timeline.log if r["kind"] == k]


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
class TestEngines:
    def test_round_time_is_barrier_plus_agg_cost(self):
        eng, _ = _run(*make_world([1.0, 0.5, 1.0 / 3.0], a_s=1.0 / 3.0))
        agg = _kind(eng, "aggregate")
        assert len(agg) == 1 and agg[0]["barrier_t_s"] == pytest.approx(30.0)
        assert agg[0]["t_s"] == pytest.approx(31.0)

    def test_straggler_dominates(self):
        eng, _ = _run(*make_world([100.0] * 19 + [10.0 / 700.0]))
        assert _kind(eng, "aggregate")[0]["barrier_t_s"] == pytest.approx(700.0)

    def test_rejected_client_skips_upload(self):
        world, w0 = make_world([1.0, 1.0], theta=1.0, up=5.0)
        eng, state = _run(world, w0)
        assert not _kind(eng, "upload_arrive")
        assert _kind(eng, "aggregate")[0]["count"] == 0
        assert np.array_equal(state.w_g.values, w0.values)

    def test_all_clients_dropped_stalls(self):
        world, w0 = make_world([1.0, 1.0], dropout=1.0, rounds=2)
        eng, state = _run(world, w0)
        kinds = [r["kind"] for r in eng.timeline.log]
        assert kinds.count("round_stalled") == 2 and "aggregate" not in kinds
        assert np.array_equal(state.w_g.values, w0.values)
        assert eng.reports[-1].failures == 2

    def test_baseline_equals_theta_zero_filtered(self):
        from paper_2503_15448_b200.config import ExperimentConfig
        from paper_2503_15448_b200.experiment import run_experiment

        cfg = ExperimentConfig.from_dict({"dataset": {"n": 1500, "d": 6, "separation": 3.0}, "num_clients": 3,
                                          "rounds": 2, "epochs": 1, "model": {"hidden_dims": [8]},
                                          "mode": "sync_baseline", "theta": 0.65, "seed": 4})
        a = run_experiment(cfg)
        b = run_experiment(cfg.with_overrides(mode="sync_filtered", theta=0.0))
        assert a.digest == b.digest and np.array_equal(a.final_params.values, b.final_params.values)

    def test_causality(self):
        from paper_2503_15448_b200.simnet import check_causality

        eng, _ = _run(*make_world([1.0, 2.0, 0.5], rounds=3, up=0.5, down=0.5))
        check_causality(eng.timeline.log)
        eng, _ = _run(*make_world([3.0, 1.0, 0.7], mode="async_filtered", rounds=2, up=0.3, down=0.4, dropout=0.2))
        check_causality(eng.timeline.log)

    def test_async_single_client_matches_sync_times(self):
        es, _ = _run(*make_world([2.0], rounds=3, up=1.0, down=1.0, a_s=0.1))
        ea, _ = _run(*make_world([2.0], mode="async_filtered", rounds=3, up=1.0, down=1.0, a_s=0.1))
        assert [r["t_s"] for r in _kind(ea, "aggregate")] == pytest.approx([r["t_s"] for r in _kind(es, "aggregate")])

    def test_async_fast_client_contributes_more(self):
        world, w0 = make_world([10.0, 1.0], mode="async_filtered", rounds=100, n_rows=10, k_min=1)
        world.horizon_s = 500.0
        eng, _ = _run(world, w0)
        done = _kind(eng, "train_done")
        fast = sum(r["client_id"] == 0 for r in done)
        slow = sum(r["client_id"] == 1 for r in done)
        assert slow > 0 and fast / slow == pytest.approx(10.0, rel=0.15)

    def test_async_budget_and_timeout(self):
        world, w0 = make_world([1.0, 1.0], mode="async_filtered", rounds=2, k_min=2)
        eng, _ = _run(world, w0)
        assert _kind(eng, "run_end")[-1]["reason"] == "budget"
        assert sum(r["count"] for r in _kind(eng, "aggregate")) == world.update_budget
        eng, _ = _run(*make_world([2.0], mode="async_filtered", rounds=2, k_min=2, timeout_s=1.0))
        trig = [r.get("trigger") for r in _kind(eng, "aggregate")]
        assert trig and all(t == "timeout" for t in trig)

    def test_async_staleness_recorded(self):
        eng, _ = _run(*make_world([5.0, 1.0], mode="async_filtered", rounds=3, k_min=1))
        st = [s for r in _kind(eng, "aggregate") for s in r["staleness"]]
        assert st and min(st) >= 0 and max(st) > 0

    def test_zero_epochs_returns_start(self):
        from paper_2503_15448_b200.client import train_local
        from paper_2503_15448_b200.model import ModelSpec, init_params

        spec = ModelSpec(input_dim=4, hidden_dims=(6,), dropout_rate=0.3)
        w0 = init_params(spec, 2)
        x = np.random.default_rng(0).normal(size=(9, 4))
        y = np.zeros(9, dtype=np.int8)
        upd = train_local(spec, _profile(), w0, x, y, 0, 4, lambda e: 0.1, seed=1)
        assert upd.steps == 0 and np.array_equal(upd.params.values, w0.values)
        with pytest.raises(ValueError):
            train_local(spec, _profile(), w0, np.zeros((0, 4)), np.zeros(0), 1, 8, lambda e: 0.1, 1)

    def test_selection_properties(self):
        from paper_2503_15448_b200.model import ParamVector
        from paper_2503_15448_b200.selection import SelectionPolicy, calculate_relevance, filter_update

        rng = np.random.default_rng(11)
        pv = lambda v: ParamVector(np.asarray(v, dtype=float), "d")
        a, b = rng.normal(size=300), rng.normal(size=300)
        s1, s2 = calculate_relevance(pv(a), pv(b)), calculate_relevance(pv(b), pv(a))
        assert s1 == s2  # symmetry
        assert calculate_relevance(pv(a * 3.5), pv(b * 0.2)) == s1  # positive-scale invariance
        assert calculate_relevance(pv([0.0, 1.0]), pv([0.0, -1.0])).aligned == 1  # zero is its own class

        class U:
            def __init__(self, p):
                self.params = p

        thetas = np.linspace(0, 1, 11)
        acc = [filter_update(U(pv(a)), pv(b), None, SelectionPolicy(theta=t))[0] for t in thetas]
        assert all(x >= y for x, y in zip(acc, acc[1:]))  # monotone in theta
        assert acc[0] and filter_update(U(pv(a)), pv(a), None, SelectionPolicy(theta=1.0))[0]
