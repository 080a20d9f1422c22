"""Host time from run_sync_round entry to the trainer launch (C4 bf16), with a
cProfile of that window (diagnostic)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import device as D  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, GlobalState  # noqa: E402

world, init = bench.build_c4_world(precision="bf16")
eng = FederationEngine(world)
st = GlobalState(round=0, w_g=init)
for _ in range(4):
    st = eng.run_sync_round(st)
torch.cuda.synchronize()
orig = D.run_trainer
T = {}


def wrapped(*a, **k):
    T["enter"] = time.perf_counter()
    out = orig(*a, **k)
    T["exit"] = time.perf_counter()
    return out


D.run_trainer = wrapped
rows = []
for rep in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = eng.run_sync_round(st)
    torch.cuda.synchronize()
    rows.append((T["enter"] - t0, T["exit"] - t0))
a = np.array(rows) * 1e6
print(f"run_trainer entered at {np.median(a[:, 0]):.1f} us, returned at {np.median(a[:, 1]):.1f} us")
pr = cProfile.Profile()
D.run_trainer = lambda *a, **k: (pr.disable(), orig(*a, **k))[1]
for rep in range(20):
    torch.cuda.synchronize()
    pr.enable()
    st = eng.run_sync_round(st)
    pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
