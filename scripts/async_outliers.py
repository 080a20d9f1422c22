"""Where do slow C4 async runs spend their wall time? cProfile per repetition (diagnostic)."""
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

cfg = dict(bench.C4_SYNC)
cfg.update({"mode": "async_filtered", "rounds": 2})
world, init = build_world(ExperimentConfig.from_dict(cfg), precision="bf16")
world.device_state()
for rep in range(int(os.environ.get("REPS", "8"))):
    torch.cuda.synchronize()
    eng = FederationEngine(world)
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    eng.run(init)
    torch.cuda.synchronize()
    pr.disable()
    wall = time.perf_counter() - t0
    print(f"rep {rep}: wall {wall:.3f}s host {eng.async_host_s}", flush=True)
    if wall > 0.25:
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(10)
        print("\n".join(s.getvalue().splitlines()[:30]), flush=True)
