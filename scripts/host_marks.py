"""Host-side phase marks of C4 bf16 sync rounds (diagnostic): host seconds
between the FederationEngine._mark points, and the device time of each
mark relative to the round's first event."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, GlobalState  # noqa: E402

world, init = bench.build_c4_world(precision="bf16")
eng = FederationEngine(world)
st = GlobalState(round=0, w_g=init)
for _ in range(4):
    st = eng.run_sync_round(st)
torch.cuda.synchronize()
rows = {}
for rep in range(8):
    eng.trace = []
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    a.record()
    h0 = time.perf_counter()
    eng._mark("start")
    st = eng.run_sync_round(st)
    eng._mark("end")
    torch.cuda.synchronize()
    for label, h, ev in eng.trace:
        rows.setdefault(label, []).append(((h - h0) * 1e6, a.elapsed_time(ev) * 1e3))
for label, v in rows.items():
    v = np.array(v)
    print(f"{label:40s} host {np.median(v[:, 0]):8.1f} us   device {np.median(v[:, 1]):8.1f} us")
