"""Host cost breakdown of device.run_trainer in C4 bf16 sync rounds (diagnostic)."""
import os
import sys
import time
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import device as D  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, GlobalState  # noqa: E402

world, init = bench.build_c4_world(precision="bf16")
eng = FederationEngine(world)
st = GlobalState(round=0, w_g=init)
for _ in range(3):
    st = eng.run_sync_round(st)
torch.cuda.synchronize()
acc = defaultdict(float)


def wrap(owner, name, label):
    f = getattr(owner, name)

    def w(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            acc[label] += time.perf_counter() - t
    setattr(owner, name, w)


rt = D.Runtime.get()
lib = rt.lib
for fn in ("fs_fill_u64", "fs_train_bf16"):
    wrap(lib, fn, fn)
for m in ("consume", "pool_buf", "static_desc"):
    wrap(D.TrainPlan, m, m)
wrap(D.Runtime, "scratch", "scratch")
wrap(D, "run_trainer", "run_trainer total")
R = 20
for _ in range(R):
    st = eng.run_sync_round(st)
torch.cuda.synchronize()
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"{k:20s} {v / R * 1e6:8.1f} us/round")
