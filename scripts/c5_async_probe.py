"""C5-style async_filtered run with the WIDE MLP (diagnostic): which engine
runs, does it finish, how fast."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200.config import ExperimentConfig  # noqa: E402
from paper_2503_15448_b200.experiment import build_world  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = dict(bench.C5_SHARE)
cfg.update({"mode": "async_filtered", "num_clients": n, "rounds": 1})
cfg["dataset"] = dict(cfg["dataset"], n=max(2000, 219176 * n // 8192))
world, init = build_world(ExperimentConfig.from_dict(cfg), precision="bf16")
world.device_state()
for rep in range(2):
    eng = FederationEngine(world)
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng.run(init)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"n={n} rep {rep}: {dt:.3f}s trainings {eng.trainings} batches {getattr(eng, 'device_batches', None)} "
          f"digest {eng.timeline.digest()} engine {getattr(eng, 'async_engine', '?')}", flush=True)
