"""Pin the CPU oracle (oracle/fl_oracle.py) against the reference's own outputs.

The golden vectors were produced by running the reference package
(tests/golden/make_golden.py); the oracle must reproduce the integer
results exactly and the float results to the reference's cross-backend
tolerance, and whole runs must replay to the identical event-log digest.
"""

import hashlib

import numpy as np
import pytest

from oracle import fl_oracle as O


def test_rng_streams_match_reference(golden):
    g = golden("rng.npz")
    for (m, cid, cyc), want in zip(g["train_seeds"], g["train_seed_out"]):
        assert O.sub_seed(int(m), "train", int(cid), int(cyc)) == int(want)
    at = 0
    for ts, e, n in g["perm_meta"]:
        n = int(n)
        got = O.sub_rng(int(ts), "shuffle", int(e)).permutation(n)
        assert np.array_equal(got, g["perm_flat"][at:at + n])
        at += n
    at = 0
    for ts, e, s, b, ms in g["mask_meta"]:
        assert O.sub_seed(int(ts), "mask", int(e), int(s)) == int(ms)
        masks = O.keep_masks((256, 128, 64), 0.3, int(b), int(ms))
        bits = np.concatenate([x.ravel() for x in masks]) > 0
        nbytes = (bits.size + 7) // 8
        assert np.array_equal(np.packbits(bits, bitorder="little"), g["mask_bits"][at:at + nbytes])
        at += nbytes


def _masks(dims, rate, rows, mseed):
    return O.keep_masks(tuple(dims[1:-1]), float(rate), rows, mseed) if mseed >= 0 else None


def test_kernels_match_reference(golden):
    k = golden("kernels.npz")
    t = 0
    while f"c{t}_dims" in k:
        dims = tuple(int(v) for v in k[f"c{t}_dims"])
        x, y, w = k[f"c{t}_x"], k[f"c{t}_y"], k[f"c{t}_w"]
        m = _masks(dims, k[f"c{t}_rate"], x.shape[0], int(k[f"c{t}_mseed"]))
        loss, grad = O.bce_grad(w, dims, x, y, m)
        assert loss == pytest.approx(float(k[f"c{t}_loss"]), rel=1e-12, abs=1e-14)
        scale = np.maximum(np.abs(k[f"c{t}_grad"]), 1.0)
        assert np.max(np.abs(grad - k[f"c{t}_grad"]) / scale) < 1e-12
        assert np.max(np.abs(O.probs(w, dims, x, m) - k[f"c{t}_fwd"])) < 1e-12
        t += 1
    t = 0
    while f"s{t}_a" in k:
        assert O.sign_matches(k[f"s{t}_a"], k[f"s{t}_b"]) == int(k[f"s{t}_count"])
        t += 1


def test_train_local_matches_reference(golden):
    tr = golden("train.npz")
    t = 0
    while f"t{t}_dims" in tr:
        dims = tuple(int(v) for v in tr[f"t{t}_dims"])
        ep, bs, seed = (int(v) for v in tr[f"t{t}_meta"])
        res = O.local_sgd(dims, float(tr[f"t{t}_rate"]), tr[f"t{t}_w0"], tr[f"t{t}_x"], tr[f"t{t}_y"], ep, bs,
                          lambda e: 0.05 * (0.9 ** e), seed)
        want = tr[f"t{t}_out"]
        assert res["steps"] == int(tr[f"t{t}_steps"])
        assert np.max(np.abs(res["params"] - want) / np.maximum(np.abs(want), 1.0)) < 1e-12
        t += 1


def test_aggregate_matches_reference_bitwise(golden):
    ag = golden("agg.npz")
    t = 0
    while f"a{t}_in" in ag:
        out = O.fedavg(list(ag[f"a{t}_in"]))
        assert np.array_equal(out, ag[f"a{t}_out"])
        t += 1


def test_world_builder_matches_reference(golden):
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world
    from tests.golden.make_golden import world_digest

    want = golden("worlds.json")
    runs = golden("runs.json")
    for name, cfg in runs.items():
        world, init = build_world(ExperimentConfig.from_dict(cfg["config"]))
        assert world_digest(world, init) == want[name], name


@pytest.mark.parametrize("name", ["sync_weight", "sync_delta_dyn", "sync_baseline", "sync_fail_ckpt",
                                  "async_fail_lost", "async_weight", "async_delta_dyn", "unsw_sync_delta"])
def test_oracle_runs_replay_reference_digest(golden, name):
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world

    runs = golden("runs.json")
    run = runs[name]
    world, init = build_world(ExperimentConfig.from_dict(run["config"]))
    sim = O.OracleFederation(world)
    wg = sim.run(init.values)
    assert sim.digest() == run["digest"]
    assert [a for _, _, a in sim.aligned_log] == run["aligned"]
    want = golden("runs_wg.npz")[name]
    assert np.max(np.abs(wg - want) / np.maximum(np.abs(want), 1.0)) < 1e-12
    for got, ref in zip(sim.reports, run["reports"]):
        assert got["accuracy"] == pytest.approx(ref["accuracy"], abs=1e-9)
        assert got["auc"] == pytest.approx(ref["auc"], abs=1e-9)
        assert got["accepted"] == ref["accepted"] and got["sgd_steps"] == ref["sgd_steps"]


def test_oracle_replays_reference_at_road_config():
    """BASELINE configs[2] (C3: 256 ROAD-shaped clients, sync_filtered,
    delta_sign, 2 rounds; tests/golden/configs.json recorded from the
    reference package): the oracle replays the digest and final model. The
    larger configs (C1, C2, C4) are checked against the CUDA path only
    (tests/test_gpu_configs.py); the oracle needs minutes per C4 round."""
    import json
    import os

    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world
    from tests.conftest import GOLDEN

    ref = json.load(open(os.path.join(GOLDEN, "configs.json")))["c3_sync"]
    want = np.load(os.path.join(GOLDEN, "configs_wg.npz"))["c3_sync_wg"]
    world, init = build_world(ExperimentConfig.from_dict(ref["config"]))
    sim = O.OracleFederation(world)
    wg = sim.run(init.values)
    assert sim.digest() == ref["digest"]
    assert np.max(np.abs(wg - want) / np.maximum(np.abs(want), 1.0)) < 1e-12


def test_world_builder_matches_reference_at_c5_scale():
    """BASELINE configs[4] world (8192 clients, alpha = 5, WIDE MLP): the
    host world builder reproduces the reference's world digest
    (tests/golden/c5_world.json, recorded from the reference package)."""
    import json
    import os

    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world
    from tests.conftest import GOLDEN
    from tests.golden.make_golden import world_digest

    ref = json.load(open(os.path.join(GOLDEN, "c5_world.json")))
    world, init = build_world(ExperimentConfig.from_dict(ref["config"]))
    assert world.num_clients == 8192 and world.spec.param_count == ref["param_count"]
    n = [wc.n for wc in world.clients]
    assert (min(n), max(n), sum(n)) == (ref["rows_min"], ref["rows_max"], ref["rows_total"])
    assert world_digest(world, init) == ref["digest"]
