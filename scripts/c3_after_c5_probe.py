"""C3 sync run times in a fresh process vs after the C5-share and C1/C2 measurements (diagnostic)."""
import os
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


def runs(tag):
    world, init = build_world(ExperimentConfig.from_dict(c3), precision="bf16")
    world.device_state()
    for rep in range(5):
        eng = FederationEngine(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        eng.run(init)
        b.record()
        torch.cuda.synchronize()
        print(f"{tag} c3 run {rep}: {a.elapsed_time(b):.2f} ms device, {1e3 * (time.perf_counter() - t0):.2f} ms host",
              flush=True)


runs("fresh")
bench.measure_c5_share("bf16", rounds=1)
runs("after c5")
print(torch.cuda.memory_stats()["num_alloc_retries"], torch.cuda.memory_reserved() / 2**30, "GiB reserved")
