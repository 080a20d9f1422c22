"""Repeated C4 async runs on one world: digest stability + time (diagnostic)."""
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
cfg = dict(bench.C4_SYNC)
cfg.update({"mode": "async_filtered", "rounds": 2})
world, init = build_world(ExperimentConfig.from_dict(cfg), precision=prec)
world.device_state()
for rep in range(int(os.environ.get("REPS", "3"))):
    torch.cuda.synchronize()
    eng = FederationEngine(world)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    eng.run(init)
    b.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: wall {time.perf_counter() - t0:.3f}s events {a.elapsed_time(b) / 1e3:.3f}s "
          f"digest {eng.timeline.digest()} host {eng.async_host_s} flushes {eng.device_batches}", flush=True)
