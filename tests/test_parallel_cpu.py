"""Client-sharded round exchange (parallel.py) on CPU with gloo, world size 2.

Each rank plays one GPU: it computes its own clients' cycle outcomes with
the CPU oracle, packs [partial FedAvg sum | aligned counts | k | diverged]
into the same buffer the CUDA path uses and all-reduces it. The reduced
results must reproduce the single-process round: identical per-client
aligned counts and accepted count, and the same global mean to float64
rounding (cross-rank re-association).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_15448_b200.parallel import RoundExchange, client_work, lpt_owner

CFG = {"num_clients": 7, "rounds": 2, "epochs": 1, "dataset": {"n": 2400, "d": 10},
       "model": {"hidden_dims": [12, 6], "dropout_rate": 0.3}, "selection_mode": "delta_sign",
       "theta": 0.5, "batch": {"policy": "dynamic", "b_ref": 16, "b_min": 8, "b_max": 64},
       "profiles": {"capacity": {"distribution": "loguniform", "low": 0.25, "high": 4.0},
                    "speed": {"distribution": "constant", "value": 50.0},
                    "up_latency": {"distribution": "constant", "value": 1.0},
                    "down_latency": {"distribution": "constant", "value": 1.0}}, "seed": 8}


def _world():
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world

    return build_world(ExperimentConfig.from_dict(CFG))


def test_lpt_owner_balances_and_is_deterministic():
    rng = np.random.default_rng(0)
    work = rng.integers(1, 1000, 1024).astype(float)
    for g in (1, 2, 4, 8):
        own = lpt_owner(work, g)
        assert np.array_equal(own, lpt_owner(work, g))
        loads = np.bincount(own, weights=work, minlength=g)
        assert loads.max() <= work.sum() / g + work.max()
        assert set(own.tolist()) == set(range(g))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, size, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    from oracle.fl_oracle import OracleFederation

    world, init = _world()
    sim = OracleFederation(world)
    owner = lpt_owner(client_work(world), size)
    mine = np.flatnonzero(owner == rank)
    w0 = init.values
    outs = [sim.cycle(int(ci), 0, 0, w0, w0 * 0.98 + 0.001) for ci in mine]
    aligned = [a for (_, _, a) in sim.aligned_log]
    M = len(w0)
    ex = RoundExchange(M, world.num_clients, torch.device("cpu"))
    acc = [o for o in outs if o["accepted"]]
    part = np.zeros(M)
    for v in sorted((o["res"]["params"] for o in acc), key=lambda v: v.tobytes()):
        part = part + v
    ex.partial_sum.copy_(torch.from_numpy(part))
    total, aligned_all, k, div = ex.reduce(mine, aligned, np.zeros(len(mine)), len(acc))
    q.put((rank, total.numpy().copy(), aligned_all, k, div))
    dist.destroy_process_group()


def test_two_rank_exchange_reproduces_single_process_round():
    from oracle.fl_oracle import OracleFederation, fedavg

    size = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(size)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    world, init = _world()
    sim = OracleFederation(world)
    outs = [sim.cycle(ci, 0, 0, init.values, init.values * 0.98 + 0.001) for ci in range(world.num_clients)]
    want_aligned = np.array([a for (_, _, a) in sim.aligned_log])
    acc = [o["res"]["params"] for o in outs if o["accepted"]]
    assert 0 < len(acc) < world.num_clients  # theta splits the clients
    want_mean = fedavg(acc)
    for rank, total, aligned_all, k, div in res:
        assert np.array_equal(aligned_all, want_aligned)
        assert k == len(acc)
        assert not div.any()
        np.testing.assert_allclose(total / k, want_mean, rtol=1e-13, atol=1e-15)
