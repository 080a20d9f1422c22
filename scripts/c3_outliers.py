"""Where do slow C3 sync runs spend their time? cProfile per run, top entries of the slowest (diagnostic)."""
import cProfile
import io
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200.config import ExperimentConfig  # noqa: E402
from paper_2503_15448_b200.experiment import build_world  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine  # noqa: E402

base = {"epochs": 5, "theta": 0.65, "seed": 1, "selection_mode": "delta_sign", "profiles": bench.C4_SYNC["profiles"],
        "model": {"hidden_dims": [256, 128, 64], "dropout_rate": 0.3}}
c3 = dict(base, num_clients=256, rounds=5, mode="sync_filtered", batch={"policy": "fixed", "size": 64},
          dataset={"kind": "synthetic", "d": 64, "samples_per_client": 256, "anomaly_frac": 0.1, "separation": 2.0,
                   "test_frac": 0.2})
world, init = build_world(ExperimentConfig.from_dict(c3), precision="bf16")
world.device_state()
res = []
for rep in range(12):
    eng = FederationEngine(world)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    eng.run(init)
    torch.cuda.synchronize()
    pr.disable()
    dt = time.perf_counter() - t0
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(8)
    res.append((dt, s.getvalue()))
    print(f"run {rep}: {1e3 * dt:.1f} ms", flush=True)
res.sort(key=lambda x: -x[0])
print(res[0][1][-2500:])
