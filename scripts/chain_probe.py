"""Critical-chain probe (diagnostic): the bf16 trainer's per-chunk-step latency
on the C4 world's longest clients, alone (one client per launch, nothing else
on the GPU) and inside a full 1024-client launch, plus the per-phase cycle
split of the lone client.

    python scripts/chain_probe.py [n_longest]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import _native as N  # noqa: E402
from paper_2503_15448_b200 import device as D  # noqa: E402
from paper_2503_15448_b200.server import train_seeds  # noqa: E402

NAMES = {0: "gather", 1: "F0 mma", 2: "F1 mma", 3: "F2 mma", 5: "F0 epi", 6: "F1 epi", 7: "F2 epi+z",
         9: "head z/dz", 11: "D3 + head upd", 12: "B0 mma", 13: "B1 mma", 14: "B2 mma",
         17: "B1 D-epi", 18: "B2 D-epi", 20: "B0 refresh", 25: "chunk end barrier",
         26: "client setup: W0 + biases", 27: "client end sync", 28: "X tile stores", 29: "mask finish",
         30: "client: write-back + claim", 31: "client setup: W1/W2",
         4: "F0 sync", 8: "F0 issue", 10: "B1 sync", 15: "B1 issue", 16: "B1 W2 upd", 19: "F1 sync",
         21: "F1 issue", 22: "B0 sync", 23: "B0 issue"}

if os.environ.get("CHAIN_C3"):  # the C3 world (256 ROAD clients, b = 64)
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world

    cfg = {"epochs": 5, "theta": 0.65, "seed": 1, "selection_mode": "delta_sign", "profiles": bench.C4_SYNC["profiles"],
           "model": {"hidden_dims": [256, 128, 64], "dropout_rate": 0.3}, "num_clients": 256, "rounds": 5,
           "mode": "sync_filtered", "batch": {"policy": "fixed", "size": 64},
           "dataset": {"kind": "synthetic", "d": 64, "samples_per_client": 256, "anomaly_frac": 0.1,
                       "separation": 2.0, "test_frac": 0.2}}
    world, init = build_world(ExperimentConfig.from_dict(cfg), precision="bf16")
else:
    world, init = bench.build_c4_world(precision="bf16")
dev = world.device_state()
rt = dev.rt
spec = world.spec
E = world.epochs
steps = dev.steps_arr
order = np.argsort(-steps, kind="stable")
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
lib = N.load()
w0 = init.device_tensor().to(torch.float32).contiguous()


def run(idx, prof=None, reps=5):
    idx = np.asarray(idx, dtype=np.int64)
    seeds = train_seeds(world.master_seed, dev.cid_arr[idx], np.zeros(len(idx), dtype=np.int32))
    lr = np.full((len(idx), E), 0.05)
    starts = np.full(len(idx), w0.data_ptr(), dtype=np.uint64)
    ts = []
    for r in range(reps):
        plan = D.TrainPlan(spec.dims, dev.shards, idx, seeds, dev.batch[idx], E, spec.dropout_rate, None, None, rt)
        plan.consume(torch.cuda.current_stream())
        torch.cuda.synchronize()
        if prof is not None and r == reps - 1:
            lib.fs_bf16_set_profile(prof.data_ptr())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        D.run_trainer(plan, lr, starts, "bf16")
        b.record()
        torch.cuda.synchronize()
        if prof is not None and r == reps - 1:
            lib.fs_bf16_set_profile(None)
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


if os.environ.get("CHAIN_SINGLE"):  # ncu target: the longest client alone, a few launches
    for _ in range(3):
        run([order[0]], reps=1)
    sys.exit(0)
print("longest clients (steps = E * steps/epoch, batch):",
      [(int(i), int(steps[i]), int(dev.batch[i])) for i in order[:k]])
for i in order[:k]:
    t = run([i])
    print(f"client {i}: alone {t * 1e3:8.1f} us, {steps[i]} steps (b={dev.batch[i]}): "
          f"{t * 1e3 / steps[i]:6.2f} us per step")
prof = torch.zeros(32, dtype=torch.int64, device="cuda")
t = run([order[0]], prof)
p = prof.cpu().numpy().astype(float)
tot = p.sum()
print(f"phase split of client {order[0]} alone ({tot / steps[order[0]]:.0f} cycles per step):")
for j in range(32):
    if p[j]:
        print(f"  {j:2d} {NAMES.get(j, '?'):28s} {100 * p[j] / tot:6.2f}%  {p[j] / steps[order[0]]:8.0f} cyc/step")
allidx = np.arange(len(dev.batch))
t_all = run(allidx)
print(f"full launch ({len(allidx)} clients): {t_all * 1e3:.1f} us")
