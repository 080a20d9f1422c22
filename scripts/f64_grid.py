"""fp64 parity trainer: C4 round trainer time vs persistent grid size (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import device as D  # noqa: E402
from paper_2503_15448_b200.server import train_seeds  # noqa: E402

world, init = bench.build_c4_world(precision="fp64")
dev = world.device_state()
spec, E = world.spec, world.epochs
w0 = init.device_tensor()
idx = np.arange(len(dev.batch))
seeds = train_seeds(world.master_seed, dev.cid_arr[idx], np.zeros(len(idx), dtype=np.int32))
lr = np.full((len(idx), E), 0.05)
starts = np.full(len(idx), w0.data_ptr(), dtype=np.uint64)
for g in [int(x) for x in (sys.argv[1:] or ["0", "148", "128", "112", "96", "74"])]:
    D.TRAIN_GRID = g
    ts = []
    for r in range(4):
        plan = D.TrainPlan(spec.dims, dev.shards, idx, seeds, dev.batch[idx], E, spec.dropout_rate, None, None, dev.rt)
        plan.consume(torch.cuda.current_stream())
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        D.run_trainer(plan, lr, starts, "fp64")
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"grid {g:4d}: {np.median(ts[1:]):7.2f} ms  ({[round(t, 2) for t in ts]})", flush=True)
