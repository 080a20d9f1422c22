"""Client-sharded sync rounds under torchrun (every rank runs the engine with
a ShardComm) against a single-process run of the same world, on rank 0.

    FS_DIST_BACKEND=gloo python -m torch.distributed.run --nproc-per-node 2 \\
        --master-addr 127.0.0.1 --master-port 29555 scripts/sharded_check.py [fp64|bf16] [mode] [selection] \\
        [c5|-] [device|native]

async engine: "device" (default) = the C++ engine's own device executor with
the all-reduce hook; "native" = ShardedAsyncExecutor (Python) under the C++ loop.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_15448_b200.config import ExperimentConfig  # noqa: E402
from paper_2503_15448_b200.experiment import build_world  # noqa: E402
from paper_2503_15448_b200.parallel import ShardComm  # noqa: E402
from paper_2503_15448_b200 import server  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
mode = sys.argv[2] if len(sys.argv) > 2 else "sync_filtered"
sel = sys.argv[3] if len(sys.argv) > 3 else "delta_sign"
engine = sys.argv[5] if len(sys.argv) > 5 else "device"
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
cfg = {"num_clients": 40, "rounds": 3, "epochs": 1, "mode": mode, "selection_mode": sel,
       "dataset": {"n": 12000, "d": 42}, "batch": {"policy": "dynamic"}, "seed": 11,
       "profiles": {"speed": {"distribution": "loguniform", "low": 20.0, "high": 200.0},
                    "capacity": {"distribution": "loguniform", "low": 0.25, "high": 4.0},
                    "up_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5},
                    "down_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5}}}
if len(sys.argv) > 4 and sys.argv[4] == "c5":
    # BASELINE configs[4]'s client population at a reduced row count: 8192
    # clients, Dirichlet alpha = 5 (alpha = 0.5 cannot partition 8192 clients),
    # UNSW MLP instead of the WIDE one (two ranks share one GPU here)
    cfg.update({"num_clients": 8192, "rounds": 2, "dataset": {"n": 60000, "d": 42}, "partition": {"alpha": 5.0},
                "batch": {"policy": "fixed", "size": 64}})
comm = ShardComm.from_env()
server._ASYNC_ENGINE = engine  # the single-process reference run below uses the same engine
world, init = build_world(ExperimentConfig.from_dict(cfg), precision=prec)
eng = FederationEngine(world, comm=comm)
st = eng.run(init)
digest = eng.timeline.digest()
wg = st.w_g.values
if comm is None or comm.rank == 0:
    world1, init1 = build_world(ExperimentConfig.from_dict(cfg), precision=prec)
    ref = FederationEngine(world1)
    st1 = ref.run(init1)
    err = float(np.max(np.abs(wg - st1.w_g.values) / np.maximum(np.abs(st1.w_g.values), 1.0)))
    same_log = digest == ref.timeline.digest()
    tol = 1e-12 if prec == "fp64" else 1e-5
    print(f"SHARDED {prec} {mode} {sel} engine={engine} ranks={comm.size if comm else 1} digest_equal={same_log} "
          f"max_rel_err={err:.3e} trainings={eng.trainings}")
    assert same_log, "sharded event log differs from the single-process run"
    assert err < tol, f"sharded global model differs ({err:.3e})"
    print("SHARDED OK")
if comm is not None:
    import torch.distributed as dist

    dist.destroy_process_group()
