"""C1 (BASELINE configs[0]: 10 UNSW clients, sync_baseline, b = 64) timing probe (diagnostic):
whole 5-round runs (CUDA events) and the longest client's trainer launch alone."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import device as D  # noqa: E402
from paper_2503_15448_b200.config import ExperimentConfig  # noqa: E402
from paper_2503_15448_b200.experiment import build_world  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, train_seeds  # noqa: E402

cfg = {"epochs": 5, "theta": 0.65, "seed": 1, "selection_mode": "weight_sign", "profiles": bench.C4_SYNC["profiles"],
       "model": {"hidden_dims": [256, 128, 64], "dropout_rate": 0.3}, "num_clients": 10, "rounds": 5,
       "mode": "sync_baseline", "dataset": bench.C4_SYNC["dataset"], "batch": {"policy": "fixed", "size": 64}}
world, init = build_world(ExperimentConfig.from_dict(cfg), precision="bf16")
dev = world.device_state()
for rep in range(3):
    eng = FederationEngine(world)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.run(init)
    b.record()
    torch.cuda.synchronize()
    print(f"run {rep}: {a.elapsed_time(b):.1f} ms for 5 rounds", flush=True)
spec, E = world.spec, world.epochs
steps = dev.steps_arr
i = int(np.argmax(steps))
w0 = init.device_tensor().to(torch.float32).contiguous()
idx = np.array([i])
seeds = train_seeds(world.master_seed, dev.cid_arr[idx], np.zeros(1, dtype=np.int32))
for rep in range(3):
    plan = D.TrainPlan(spec.dims, dev.shards, idx, seeds, dev.batch[idx], E, spec.dropout_rate, None, None, dev.rt)
    plan.consume(torch.cuda.current_stream())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    D.run_trainer(plan, np.full((1, E), 0.05), np.array([w0.data_ptr()], dtype=np.uint64), "bf16")
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b)
    print(f"client {i} alone: {t:.2f} ms, {steps[i]} steps, {t * 1e3 / steps[i]:.2f} us/step", flush=True)
