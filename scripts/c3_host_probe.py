"""C3 sync: per-round host time split (marks) and cProfile of whole runs (diagnostic)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
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
for _ in range(3):
    FederationEngine(world).run(init)
torch.cuda.synchronize()
eng = FederationEngine(world)
eng.trace = []
t0 = time.perf_counter()
eng._mark("start")
eng.run(init)
torch.cuda.synchronize()
last = t0
for label, h, ev in eng.trace:
    print(f"{label:40s} +{1e6 * (h - last):9.1f} us")
    last = h
print(f"total {1e3 * (time.perf_counter() - t0):.2f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    FederationEngine(world).run(init)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
