"""Parity of the CUDA path against the reference (golden vectors) and the oracle.

Bars: bit-exact for integer/index work (seeds, permutations, mask bits,
alignment counts, aggregation order and the event-log digest); float64
results within 1e-12 relative (the reference's own compiled-vs-numpy
backends differ by up to ~3e-16); aggregation bitwise for equal inputs.
"""

import numpy as np
import pytest
import torch

from tests.conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

RUN_NAMES = ["sync_weight", "sync_delta_dyn", "sync_baseline", "sync_fail_ckpt",
             "async_fail_lost", "async_weight", "async_delta_dyn", "unsw_sync_delta"]


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))) if a.size else 0.0


# --------------------------------------------------------------------- K1-K3
def test_rng_kernels_bit_exact(golden):
    from paper_2503_15448_b200 import device as D
    from paper_2503_15448_b200.model import ModelSpec, dropout_mask_bits

    rt = D.Runtime.get()
    g = golden("rng.npz")
    meta = g["train_seeds"]
    for m in np.unique(meta[:, 0]):
        sel = meta[:, 0] == m
        cid = rt.h2d(meta[sel, 1].astype(np.int32))
        cyc = rt.h2d(meta[sel, 2].astype(np.int32))
        out = torch.empty(int(sel.sum()), dtype=torch.int64, device=rt.device)
        rt.call(rt.lib.fs_train_seeds(int(m), cid.data_ptr(), cyc.data_ptr(), int(sel.sum()), out.data_ptr(),
                                      rt.stream), "seeds")
        assert np.array_equal(out.cpu().numpy().view(np.uint64), g["train_seed_out"][sel])

    at = 0
    for ts, e, n in g["perm_meta"]:
        n, e = int(n), int(e)
        seeds = rt.h2d(np.array([ts], dtype=np.uint64).view(np.int64))
        nr = rt.h2d(np.array([n], dtype=np.int32))
        off = rt.h2d(np.array([0], dtype=np.int64))
        perm = torch.empty(n * (e + 1), dtype=torch.int32, device=rt.device)
        rt.call(rt.lib.fs_shuffle_perms(seeds.data_ptr(), nr.data_ptr(), off.data_ptr(), 1, e + 1, n,
                                        perm.data_ptr(), rt.stream), "perms")
        assert np.array_equal(perm.cpu().numpy()[e * n:(e + 1) * n], g["perm_flat"][at:at + n])
        at += n

    spec = ModelSpec(input_dim=42, hidden_dims=(256, 128, 64), dropout_rate=0.3)
    at = 0
    for ts, e, s, b, ms in g["mask_meta"]:
        words = dropout_mask_bits(spec, int(b), int(ms)).cpu().numpy().view(np.uint32)
        nbits = int(b) * 448
        bits = ((words[:, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool).ravel()[:nbits]
        nbytes = (nbits + 7) // 8
        assert np.array_equal(np.packbits(bits, bitorder="little"), g["mask_bits"][at:at + nbytes])
        at += nbytes


# --------------------------------------------------------------------- backend kernels
def test_backend_kernels_match_reference(golden):
    from paper_2503_15448_b200.backends import get_backend
    from oracle.fl_oracle import keep_masks

    be = get_backend()
    k = golden("kernels.npz")
    t = 0
    while f"c{t}_dims" in k:
        dims = tuple(int(v) for v in k[f"c{t}_dims"])
        x, y, w = k[f"c{t}_x"], k[f"c{t}_y"], k[f"c{t}_w"]
        ms = int(k[f"c{t}_mseed"])
        masks = keep_masks(dims[1:-1], float(k[f"c{t}_rate"]), x.shape[0], ms) if ms >= 0 else None
        loss, grad = be.loss_and_grad(w, dims, x, y, masks)
        assert loss == pytest.approx(float(k[f"c{t}_loss"]), rel=1e-12, abs=1e-14)
        assert rel_err(grad, k[f"c{t}_grad"]) < 1e-12
        assert np.max(np.abs(be.forward(w, dims, x, masks) - k[f"c{t}_fwd"])) < 1e-12
        t += 1
    t = 0
    while f"s{t}_a" in k:
        assert be.sign_align_count(k[f"s{t}_a"], k[f"s{t}_b"]) == int(k[f"s{t}_count"])
        t += 1


def test_sign_align_edge_cases():
    from paper_2503_15448_b200.backends import get_backend
    from paper_2503_15448_b200.model import ParamVector
    from paper_2503_15448_b200.selection import calculate_relevance

    be = get_backend()
    assert be.sign_align_count(np.array([-0.0, 0.0, 1.0, -1.0]), np.array([0.0, -0.0, 2.0, -3.0])) == 4
    assert be.sign_align_count(np.array([1.0]), np.array([-1.0])) == 0
    with pytest.raises(ValueError):
        be.sign_align_count(np.ones(3), np.ones(4))
    # reference known answers (tests/test_selection.py:45-54, 86-106)
    pv = lambda v: ParamVector(np.asarray(v, dtype=float), "d")
    assert calculate_relevance(pv([1, -1, 1, -1]), pv([1, 1, -1, -1])).ratio == 0.5
    s = calculate_relevance(pv([2.0, -2.0, 0.5, -0.5]), pv([1.0, -1.0, 1.0, -1.0]), pv([0.0] * 4), "delta_sign")
    assert s.aligned == 2
    with pytest.raises(ValueError):
        calculate_relevance(pv([2.0]), pv([1.0]), None, "delta_sign")
    from paper_2503_15448_b200.selection import SelectionPolicy, filter_update

    class _U:
        def __init__(self, p):
            self.params = p

    b = np.ones(20)
    b[13:] = -1.0
    ok, sc = filter_update(_U(pv(np.ones(20))), pv(b), None, SelectionPolicy(theta=0.65))
    assert sc.ratio == 0.65 and ok  # inclusive boundary 13/20
    # odd lengths / unaligned starts / large M across the vector path
    rng = np.random.default_rng(4)
    for n in (1, 2, 3, 1023, 4097, 52225, 300001):
        a = np.round(rng.normal(size=n), 1)
        b = np.round(rng.normal(size=n), 1)
        assert be.sign_align_count(a, b) == int(np.count_nonzero(np.sign(a) == np.sign(b)))
        assert be.sign_align_count(a[1:], b[1:]) == int(np.count_nonzero(np.sign(a[1:]) == np.sign(b[1:])))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("mode", ["weight_sign", "delta_sign"])
def test_sign_align_shared_matches_numpy(dtype, mode):
    from paper_2503_15448_b200 import device as D

    rt = D.Runtime.get()
    rng = np.random.default_rng(7)
    for n, M in ((1, 1), (3, 5), (7, 1023), (13, 52225), (6, 100003)):
        ld = (M + 31) // 32 * 32
        W = torch.tensor(np.round(rng.normal(size=(n, ld)), 1), dtype=dtype, device="cuda")[:, :M]
        g = torch.tensor(np.round(rng.normal(size=M), 1), dtype=dtype, device="cuda")
        p = torch.tensor(np.round(rng.normal(size=M), 1), dtype=dtype, device="cuda")
        rows = W.data_ptr() + np.arange(n, dtype=np.uint64) * np.uint64(ld * W.element_size())
        got = D.align_shared(rows, g, p if mode == "delta_sign" else None, M, mode, rt).cpu().numpy()
        Wn, gn, pn = W.cpu().double().numpy(), g.cpu().double().numpy(), p.cpu().double().numpy()
        if mode == "weight_sign":
            want = [(np.sign(Wn[i]) == np.sign(gn)).sum() for i in range(n)]
        else:
            want = [(np.sign(Wn[i] - gn) == np.sign(gn - pn)).sum() for i in range(n)]
        assert list(got) == [int(x) for x in want], (n, M)


def test_aggregate_bitwise(golden):
    from paper_2503_15448_b200.model import ParamVector
    from paper_2503_15448_b200.server import aggregate

    ag = golden("agg.npz")
    t = 0
    while f"a{t}_in" in ag:
        vecs = [ParamVector(v, "d") for v in ag[f"a{t}_in"]]
        assert np.array_equal(aggregate(vecs).values, ag[f"a{t}_out"])
        rev = aggregate(vecs[::-1]).values
        assert np.array_equal(rev, ag[f"a{t}_out"])
        t += 1
    assert aggregate([]) is None
    with pytest.raises(ValueError):
        aggregate([ParamVector(np.ones(1), "d"), ParamVector(np.ones(2), "d")])


# --------------------------------------------------------------------- trainer
def test_train_local_matches_reference(golden):
    from paper_2503_15448_b200.client import ClientProfile, train_local
    from paper_2503_15448_b200.model import ModelSpec, ParamVector

    tr = golden("train.npz")
    prof = ClientProfile(id=0, speed=50.0, up_latency_s=1.0, down_latency_s=1.0, capacity=1.0)
    t = 0
    while f"t{t}_dims" in tr:
        dims = tuple(int(v) for v in tr[f"t{t}_dims"])
        spec = ModelSpec(input_dim=dims[0], hidden_dims=dims[1:-1], dropout_rate=float(tr[f"t{t}_rate"]))
        ep, bs, seed = (int(v) for v in tr[f"t{t}_meta"])
        w0 = ParamVector(tr[f"t{t}_w0"], spec.digest())
        upd = train_local(spec, prof, w0, tr[f"t{t}_x"], tr[f"t{t}_y"], ep, bs, lambda e: 0.05 * (0.9 ** e), seed)
        assert upd.steps == int(tr[f"t{t}_steps"])
        assert rel_err(upd.params.values, tr[f"t{t}_out"]) < 1e-12
        t += 1


def _small():
    from paper_2503_15448_b200.model import ModelSpec, init_params

    spec = ModelSpec(input_dim=4, hidden_dims=(8, 5), dropout_rate=0.3)
    rng = np.random.default_rng(0)
    return spec, init_params(spec, 3), rng.normal(size=(40, 4)), rng.integers(0, 2, 40).astype(np.int8)


def test_train_local_equals_fold_of_loss_and_grad_bitwise():
    # reference tests/test_client.py:83-120: batched trainer == per-step API
    from paper_2503_15448_b200.client import ClientProfile, batch_count, train_local
    from paper_2503_15448_b200.model import Batch, loss_and_grad, sgd_step
    from paper_2503_15448_b200.rng import derive_rng, derive_seed

    spec, w0, x, y = _small()
    prof = ClientProfile(id=0, speed=50.0, up_latency_s=1.0, down_latency_s=1.0, capacity=1.0)
    epochs, bs, lr, seed = 2, 16, 0.05, 11
    upd = train_local(spec, prof, w0, x, y, epochs, bs, lambda e: lr, seed=seed)
    params = w0
    for e in range(epochs):
        perm = derive_rng(seed, "shuffle", e).permutation(40)
        for b in range(batch_count(40, bs)):
            idx = perm[b * bs:(b + 1) * bs]
            _, g = loss_and_grad(spec, params, Batch(x[idx], y[idx].astype(np.float64)),
                                 dropout_seed=derive_seed(seed, "mask", e, b))
            params = sgd_step(params, g, lr)
    assert np.array_equal(upd.params.values, params.values)


def test_stop_resume_bitwise():
    # reference tests/test_client.py:122-156
    from paper_2503_15448_b200.client import ClientProfile, TrainingProgress, train_local

    spec, w0, x, y = _small()
    prof = ClientProfile(id=0, speed=50.0, up_latency_s=1.0, down_latency_s=1.0, capacity=1.0)
    full = train_local(spec, prof, w0, x, y, 3, 8, lambda e: 0.1, seed=13)
    for cut in (1, 4, 7, full.steps - 1):
        part = train_local(spec, prof, w0, x, y, 3, 8, lambda e: 0.1, seed=13, stop_after_steps=cut)
        assert isinstance(part, TrainingProgress) and part.steps_done == cut
        res = train_local(spec, prof, w0, x, y, 3, 8, lambda e: 0.1, seed=13, resume=part)
        assert np.array_equal(res.params.values, full.params.values)
        assert res.steps == full.steps


def test_divergence_raises():
    from paper_2503_15448_b200.client import ClientProfile, train_local
    from paper_2503_15448_b200.model import ParamVector, TrainingDivergedError

    spec, w0, x, y = _small()
    prof = ClientProfile(id=0, speed=50.0, up_latency_s=1.0, down_latency_s=1.0, capacity=1.0)
    big = ParamVector(w0.values * 1e300, spec.digest())
    with pytest.raises(TrainingDivergedError):
        train_local(spec, prof, big, x * 1e10, y, 1, 8, lambda e: 1.0, seed=1)


# --------------------------------------------------------------------- eval
def test_eval_metrics_match_oracle():
    from oracle.fl_oracle import acc_auc
    from paper_2503_15448_b200.metrics import evaluate

    rng = np.random.default_rng(9)
    for n in (2, 17, 1000, 43835):
        s = np.round(rng.random(n), 3)  # heavy ties
        s[: n // 10] = 1.0
        lab = rng.integers(0, 2, n).astype(np.int8)
        lab[0], lab[-1] = 0, 1
        res = evaluate(s, lab)
        acc, auc = acc_auc(s, lab)
        assert res.accuracy == acc and res.auc == auc


# --------------------------------------------------------------------- engines
@pytest.mark.parametrize("name", RUN_NAMES)
def test_engine_replays_reference_digest(golden, name):
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world
    from paper_2503_15448_b200.server import FederationEngine

    run = golden("runs.json")[name]
    world, init = build_world(ExperimentConfig.from_dict(run["config"]))
    eng = FederationEngine(world)
    state = eng.run(init)
    assert eng.timeline.digest() == run["digest"]
    want = golden("runs_wg.npz")[name]
    assert rel_err(state.w_g.values, want) < 1e-12
    for got, ref in zip(eng.reports, run["reports"]):
        rec = got.to_record()
        for key in ("accepted", "rejected", "failures", "updates", "aggregations", "sgd_steps", "round"):
            assert rec[key] == ref[key], key
        assert rec["accuracy"] == pytest.approx(ref["accuracy"], abs=1e-9)
        assert rec["auc"] == pytest.approx(ref["auc"], abs=1e-9)


def test_engine_matches_oracle_at_unsw_shape():
    """Teacher-free end-to-end check at the UNSW MLP shape (fp64 mode)."""
    from oracle.fl_oracle import OracleFederation
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world
    from paper_2503_15448_b200.server import FederationEngine

    cfg = {"num_clients": 24, "rounds": 2, "epochs": 1, "dataset": {"n": 20000, "d": 42},
           "mode": "async_filtered", "selection_mode": "delta_sign",
           "batch": {"policy": "dynamic"}, "seed": 4,
           "profiles": {"speed": {"distribution": "loguniform", "low": 20.0, "high": 200.0},
                        "capacity": {"distribution": "loguniform", "low": 0.25, "high": 4.0},
                        "up_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5},
                        "down_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5}}}
    world, init = build_world(ExperimentConfig.from_dict(cfg))
    eng = FederationEngine(world)
    st = eng.run(init)
    sim = OracleFederation(world)
    wg = sim.run(init.values)
    assert eng.timeline.digest() == sim.digest()
    assert rel_err(st.w_g.values, wg) < 1e-12


@pytest.mark.parametrize("name", ["async_fail_lost", "async_weight", "async_delta_dyn"])
@pytest.mark.parametrize("engine", ["device", "native", "python"])
def test_async_engines_agree(golden, monkeypatch, name, engine):
    """The C++ event loop with its C++ device executor ("device", default),
    with the Python executor ("native") and the Python event loop
    ("python") replay the reference digest and the same global model bitwise."""
    from paper_2503_15448_b200 import server
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world

    monkeypatch.setattr(server, "_ASYNC_ENGINE", engine)
    run = golden("runs.json")[name]
    world, init = build_world(ExperimentConfig.from_dict(run["config"]))
    eng = server.FederationEngine(world)
    state = eng.run(init)
    assert eng.timeline.digest() == run["digest"]
    want = golden("runs_wg.npz")[name]
    assert rel_err(state.w_g.values, want) < 1e-12
    assert [r.accepted for r in eng.reports] == [r["accepted"] for r in run["reports"]]
    assert [r.transfer_s for r in eng.reports] == pytest.approx([r["transfer_s"] for r in run["reports"]], abs=0)
    assert len(state.history) == sum(1 for r in eng.timeline.log if r["kind"] == "aggregate")


@pytest.mark.parametrize("extra", [{}, {"dropout_rate": 0.3, "checkpoint": {"enabled": True, "total_time_s": 60.0,
                                                                           "recovery_s": 2.0}},
                                   {"dropout_rate": 0.3}, {"aggregation": {"k_min": 1}}],
                         ids=["plain", "fail_ckpt", "fail_lost", "k_min1"])
def test_async_engines_agree_bf16(extra):
    """bf16 mode: the three async engines make the same decisions and produce
    the same float32 global model bitwise (same kernels, same order)."""
    from paper_2503_15448_b200 import server
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world

    cfg = {"num_clients": 48, "rounds": 2, "epochs": 1, "dataset": {"n": 20000, "d": 42},
           "mode": "async_filtered", "selection_mode": "delta_sign", "batch": {"policy": "dynamic"}, "seed": 6,
           "profiles": {"speed": {"distribution": "loguniform", "low": 20.0, "high": 200.0},
                        "capacity": {"distribution": "loguniform", "low": 0.25, "high": 4.0},
                        "up_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5},
                        "down_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5}}}
    cfg.update(extra)
    out = {}
    saved = server._ASYNC_ENGINE
    try:
        for engine in ("device", "native", "python"):
            server._ASYNC_ENGINE = engine
            world, init = build_world(ExperimentConfig.from_dict(cfg), precision="bf16")
            eng = server.FederationEngine(world)
            st = eng.run(init)
            out[engine] = (eng.timeline.digest(), st.w_g.values.copy())
    finally:
        server._ASYNC_ENGINE = saved
    assert out["device"][0] == out["native"][0] == out["python"][0]
    assert np.array_equal(out["device"][1], out["native"][1])
    assert np.array_equal(out["device"][1], out["python"][1])


@pytest.mark.parametrize("mode", ["sync_filtered", "async_filtered"])
def test_engine_matches_oracle_at_road_shape(mode):
    """C3's shape (ROAD CAN windows: d = 64, 256 samples per client, b = 64,
    delta_sign) in fp64 parity mode: digest and global model vs the oracle."""
    from oracle.fl_oracle import OracleFederation
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world
    from paper_2503_15448_b200.server import FederationEngine

    cfg = {"num_clients": 16, "rounds": 2, "epochs": 1, "mode": mode, "selection_mode": "delta_sign", "seed": 7,
           "dataset": {"kind": "synthetic", "d": 64, "samples_per_client": 256, "anomaly_frac": 0.1,
                       "separation": 2.0, "test_frac": 0.2},
           "batch": {"policy": "fixed", "size": 64},
           "profiles": {"speed": {"distribution": "loguniform", "low": 20.0, "high": 200.0},
                        "up_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5},
                        "down_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5}}}
    world, init = build_world(ExperimentConfig.from_dict(cfg))
    eng = FederationEngine(world)
    st = eng.run(init)
    sim = OracleFederation(world)
    wg = sim.run(init.values)
    assert eng.timeline.digest() == sim.digest()
    assert rel_err(st.w_g.values, wg) < 1e-12


@pytest.mark.parametrize("prec,mode,sel,shape,engine", [("fp64", "sync_filtered", "delta_sign", "-", "device"),
                                                        ("bf16", "sync_filtered", "delta_sign", "-", "device"),
                                                        ("fp64", "async_filtered", "weight_sign", "-", "device"),
                                                        ("bf16", "async_filtered", "weight_sign", "-", "device"),
                                                        ("bf16", "async_filtered", "delta_sign", "-", "device"),
                                                        ("fp64", "async_filtered", "weight_sign", "-", "native"),
                                                        ("bf16", "async_filtered", "weight_sign", "-", "native"),
                                                        ("fp64", "sync_filtered", "delta_sign", "c5", "device"),
                                                        ("bf16", "sync_filtered", "delta_sign", "c5", "device")])
def test_client_sharded_rounds_match_single_process(prec, mode, sel, shape, engine):
    """Two ranks (sharing the one GPU over gloo) run the client-sharded engines
    (parallel.py ownership; sync: selection, partial sum, packing and one
    all-reduce per round on the device; async: one all-reduce of the outcomes
    per flush and of the job partial sums — "device": inside the C++ engine's
    own executor through its exchange hook, "native": ShardedAsyncExecutor)
    and reproduce the single-process event log and global model; "c5": 8192
    clients at Dirichlet alpha 5."""
    import os
    import socket
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, FS_DIST_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2", "--master-addr",
                          "127.0.0.1", "--master-port", str(port), os.path.join(root, "scripts", "sharded_check.py"),
                          prec, mode, sel, shape, engine], env=env, capture_output=True, text=True, timeout=900, cwd=root)
    assert "SHARDED OK" in out.stdout, out.stdout[-2000:] + out.stderr[-3000:]


def test_engine_keeps_caller_vectors_and_checkpoints_intact(monkeypatch):
    """A bf16 run does not turn the caller's float64 vector into float32
    (device_tensor() stays float64, values unchanged); every global
    checkpoint keeps the model of its round although older ones move to host
    memory once the HBM budget is exceeded; a checkpoint is a separate vector
    from the engine state."""
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world
    from paper_2503_15448_b200 import server as S
    from paper_2503_15448_b200.server import FederationEngine, GlobalState

    monkeypatch.setattr(S._HostArchive, "DEVICE_BUDGET", 1)  # spill everything the next round does not read
    cfg = {"num_clients": 12, "rounds": 4, "epochs": 1, "selection_mode": "delta_sign", "seed": 4,
           "dataset": {"n": 4000, "d": 42}, "model": {"hidden_dims": [256, 128, 64], "dropout_rate": 0.3}}
    world, initial = build_world(ExperimentConfig.from_dict(cfg), precision="bf16")
    before = initial.values.copy()
    assert initial.device_tensor().dtype == torch.float64
    eng = FederationEngine(world)
    st = GlobalState(round=0, w_g=initial)
    seen = []
    for _ in range(4):
        st = eng.run_sync_round(st)
        seen.append(st.w_g.values.copy())
    assert initial.device_tensor().dtype == torch.float64
    assert np.array_equal(initial.values, before)
    cps = eng.global_checkpoints
    assert [c.round for c in cps] == [0, 1, 2, 3]
    # with the HBM budget exhausted only the newest stays; the others were
    # spilled during the following rounds' trainers (the state keeps its own refs)
    assert [c.params.is_on_device for c in cps] == [False, False, True, True]
    for c, want in zip(cps, seen):
        assert np.array_equal(c.params.values, want)
    assert cps[-1].params is not st.w_g
    st.w_g.values = np.zeros_like(seen[-1])  # replacing the state's values leaves the checkpoint alone
    assert np.array_equal(cps[-1].params.values, seen[-1])


def test_run_experiment_writes_reference_run_directory(tmp_path):
    """run_experiment(config, out_dir) writes the reference's run directory
    (config.json, events.jsonl, rounds.jsonl, summary.csv, run_meta.json,
    checkpoints/ with MANIFEST.json) and replay_run reproduces it."""
    import json
    import os

    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import params_digest, replay_run, run_experiment
    from paper_2503_15448_b200.fault import read_checkpoint_file
    from paper_2503_15448_b200.simnet import log_digest

    cfg = ExperimentConfig.from_dict({"num_clients": 6, "rounds": 2, "epochs": 1, "dataset": {"n": 1500, "d": 12},
                                      "model": {"hidden_dims": [16, 8], "dropout_rate": 0.3}, "seed": 3})
    res = run_experiment(cfg, str(tmp_path))
    names = set(os.listdir(tmp_path))
    assert {"config.json", "events.jsonl", "rounds.jsonl", "summary.csv", "run_meta.json", "checkpoints"} <= names
    meta = json.load(open(tmp_path / "run_meta.json"))
    assert meta["digest"] == res.digest and meta["backend"] == "b200"
    events = [json.loads(x) for x in open(tmp_path / "events.jsonl")]
    assert log_digest(events) == res.digest
    assert res.summary["rounds"] == 2 and "accuracy" in res.summary
    ck_dir = tmp_path / "checkpoints"
    files = [f for f in os.listdir(ck_dir) if f.endswith(".ckpt")]
    assert len(files) == 1 and "MANIFEST.json" in os.listdir(ck_dir)
    ck = read_checkpoint_file(str(ck_dir / files[0]))
    assert params_digest(ck.params) == meta["params_digest"] == params_digest(res.final_params)
    ok, report = replay_run(str(tmp_path))
    assert ok, report


@pytest.mark.parametrize("n", [1, 2, 3, 7, 64, 511, 1000, 1659, 5000, 65536, 70001])
def test_shuffle_perms_match_numpy_permutation(n):
    """K2 (fs_shuffle_perms: the 16-bit shared-memory kernel up to 65536 rows,
    the int32 one above) equals numpy's derive_rng(seed, "shuffle", e).permutation(n)
    (client.py:136) for every epoch, including the batch-boundary rejection
    paths of the buffered 32-bit draw stream."""
    from paper_2503_15448_b200 import device as D
    from paper_2503_15448_b200.rng import derive_rng

    rt = D.Runtime.get()
    epochs = 3
    seeds_h = np.array([0x9E3779B97F4A7C15 + n, 12345 + 7 * n], dtype=np.uint64)
    sizes = np.array([n, max(n // 3, 1)], dtype=np.int32)
    off_h = np.array([0, epochs * n], dtype=np.int64)
    seeds, nr, off = rt.h2d(seeds_h.view(np.int64)), rt.h2d(sizes), rt.h2d(off_h)
    perm = torch.empty(int(epochs * sizes.sum()), dtype=torch.int32, device=rt.device)
    rt.call(rt.lib.fs_shuffle_perms(seeds.data_ptr(), nr.data_ptr(), off.data_ptr(), 2, epochs, int(sizes.max()),
                                    perm.data_ptr(), rt.stream), "perms")
    got = perm.cpu().numpy()
    for r in range(2):
        for e in range(epochs):
            want = derive_rng(int(seeds_h[r]), "shuffle", e).permutation(int(sizes[r]))
            at = int(off_h[r]) + e * int(sizes[r])
            assert np.array_equal(got[at:at + int(sizes[r])], want), (r, e)
