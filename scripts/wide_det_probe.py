"""Determinism of WIDE-MLP runs across repetitions in one process (diagnostic)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200.config import ExperimentConfig  # noqa: E402
from paper_2503_15448_b200.experiment import build_world  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine  # noqa: E402

mode, n = sys.argv[1], int(sys.argv[2])
cfg = dict(bench.C5_SHARE)
cfg.update({"mode": mode, "num_clients": n, "rounds": 2})
cfg["dataset"] = dict(cfg["dataset"], n=max(2000, 219176 * n // 8192))
world, init = build_world(ExperimentConfig.from_dict(cfg), precision="bf16")
world.device_state()
out = []
for rep in range(3):
    eng = FederationEngine(world)
    st = eng.run(init)
    torch.cuda.synchronize()
    out.append((eng.timeline.digest(), float(abs(st.w_g.values).sum())))
print(mode, n, os.environ.get("FS_ASYNC_ENGINE", "device"), os.environ.get("FS_ASYNC_BATCH_WAIT", "0"), out, flush=True)
