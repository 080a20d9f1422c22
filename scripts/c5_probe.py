"""C5 (BASELINE configs[4]) per-GPU share on one B200: WIDE MLP 42-1024x4-1,
1024 clients (the 1/8 of 8192 one GPU owns at 8 GPUs), UNSW-shaped data scaled to
keep C5's ~21 rows per client, Dirichlet alpha = 5, b = 64, delta_sign, E = 5.
Times sync_filtered rounds and an async_filtered window (diagnostic)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_15448_b200 import device as D  # noqa: E402
from paper_2503_15448_b200.config import ExperimentConfig  # noqa: E402
from paper_2503_15448_b200.experiment import build_world  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, GlobalState  # noqa: E402

clients = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
cfg = {"num_clients": clients, "rounds": 3, "epochs": 5, "mode": "sync_filtered", "selection_mode": "delta_sign",
       "theta": 0.65, "seed": 1,
       "dataset": {"kind": "synthetic", "n": 219176 * clients // 8192, "d": 42, "anomaly_frac": 0.3,
                   "separation": 4.0, "test_frac": 0.2},
       "partition": {"alpha": 5.0},
       "model": {"hidden_dims": [1024, 1024, 1024, 1024], "dropout_rate": 0.3},
       "batch": {"policy": "fixed", "size": 64},
       "profiles": {"speed": {"distribution": "loguniform", "low": 20.0, "high": 200.0},
                    "up_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5},
                    "down_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5}}}
t0 = time.perf_counter()
world, init = build_world(ExperimentConfig.from_dict(cfg), precision=prec)
world.device_state()
print(f"world built in {time.perf_counter() - t0:.1f}s; rows/client {sum(wc.n for wc in world.clients) / clients:.1f}",
      flush=True)
eng = FederationEngine(world)
st = GlobalState(round=0, w_g=init)
st = eng.run_sync_round(st)  # warm-up
torch.cuda.synchronize()
D.Runtime.timer = D.KernelTimer()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(2):
    st = eng.run_sync_round(st)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 2
ks = D.Runtime.timer.summary()
D.Runtime.timer = None
tr = ks.get("train", {})
out = {"clients": clients, "precision": prec, "sync_ms_per_round": ms, "sync_rounds_per_s": 1000 / ms,
       "client_updates_per_s": clients * 1000 / ms,
       "train_ms": tr.get("mean_ms"), "train_tflops": tr.get("work_per_launch", 0) / (tr.get("mean_ms", 1) * 1e-3) / 1e12,
       "kernels": {k: v["mean_ms"] for k, v in ks.items()}}
print(json.dumps(out), flush=True)
cfg.update({"mode": "async_filtered", "rounds": 1})
world2, init2 = build_world(ExperimentConfig.from_dict(cfg), precision=prec)
world2.device_state()
torch.cuda.synchronize()
eng2 = FederationEngine(world2)
t0 = time.perf_counter()
eng2.run(init2)
torch.cuda.synchronize()
sec = time.perf_counter() - t0
print(json.dumps({"async_window_s": sec, "async_rounds_per_s": 1 / sec, "trainings": eng2.trainings,
                  "flushes": eng2.device_batches, "client_updates_per_s": eng2.trainings / sec}), flush=True)
