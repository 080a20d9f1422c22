"""C4 async (full adaptive framework) on one GPU: windows/s, trainings, flushes."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200.config import ExperimentConfig  # noqa: E402
from paper_2503_15448_b200.experiment import build_world  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = dict(bench.C4_SYNC)
cfg.update({"mode": "async_filtered", "rounds": rounds})
world, init = build_world(ExperimentConfig.from_dict(cfg), precision=prec)
world.device_state()
torch.cuda.synchronize()
eng = FederationEngine(world)
t0 = time.perf_counter()
st = eng.run(init)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{prec}: {rounds} windows in {dt:.2f} s -> {rounds / dt:.3f} rounds/s, trainings {eng.trainings}, "
      f"flushes {eng.device_batches}, events {len(eng.timeline.log)}, digest {eng.timeline.digest()}")
print("host s (prep, wait, post):", getattr(eng, "async_host_s", None))
