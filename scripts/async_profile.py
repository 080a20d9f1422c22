"""Where the C4 async engine's time goes: trainer GPU time vs host (diagnostic)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import device as D  # noqa: E402
from paper_2503_15448_b200.config import ExperimentConfig  # noqa: E402
from paper_2503_15448_b200.experiment import build_world  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine  # noqa: E402

cfg = dict(bench.C4_SYNC)
cfg.update({"mode": "async_filtered", "rounds": 1})
world, init = build_world(ExperimentConfig.from_dict(cfg), precision="bf16")
world.device_state()
FederationEngine(world).run(init)  # warm
torch.cuda.synchronize()
D.Runtime.timer = D.KernelTimer()
eng = FederationEngine(world)
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
eng.run(init)
torch.cuda.synchronize()
pr.disable()
wall = time.perf_counter() - t0
ks = D.Runtime.timer.summary()
print(f"wall {wall:.3f} s, trainings {eng.trainings}, flushes {eng.device_batches}")
for k, v in ks.items():
    print(f"  {k}: {v['launches']} launches, {v['total_ms']:.1f} ms total, mean {v['mean_ms']:.3f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
