"""K2 (shuffles) and K3 (dropout bits) of the C4 round plan: alone on an
idle GPU, and concurrent with the trainer (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import device as D  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, GlobalState, train_seeds  # noqa: E402

world, init = bench.build_c4_world(precision="bf16")
eng = FederationEngine(world)
state = GlobalState(round=0, w_g=init)
for _ in range(3):
    state = eng.run_sync_round(state)
torch.cuda.synchronize()
dev = world.device_state()
rt = dev.rt
idx = np.arange(world.num_clients)
seeds = train_seeds(world.master_seed, dev.cid_arr[idx], np.full(len(idx), 7, dtype=np.int32))
plan = D.TrainPlan(world.spec.dims, dev.shards, idx, seeds, dev.batch[idx], world.epochs, world.spec.dropout_rate,
                   rt=rt)
torch.cuda.synchronize()
lib, s = rt.lib, torch.cuda.current_stream().cuda_stream
n = plan.n
print("max rows", int(dev.shards.n_rows.max()), "sum rows", int(dev.shards.n_rows.sum()), "bits words", plan.bits.numel())


def timed(fn, reps=5):
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out))


k2 = lambda: lib.fs_shuffle_perms(plan.seeds_p, plan.n_rows_p, plan.perm_off_p, n, plan.epochs,  # noqa: E731
                                  int(dev.shards.n_rows.max()), plan.perm.data_ptr(), s)
k3 = lambda: lib.fs_dropout_bits(plan.seeds_p, plan.n_rows_p, plan.batch_p, plan.mask_off_p, n,  # noqa: E731
                                 plan.epochs, plan.sum_hidden, 1.0 - plan.dropout_rate, plan.bits.data_ptr(), s)
print(f"K2 alone {timed(k2):.3f} ms   K3 alone {timed(k3):.3f} ms")
