"""C5 share sync rounds (diagnostic): per-round device time and the host /
device time of each FederationEngine._mark point, for rounds 1..4 (round 0
is the warm-up, unscored under delta_sign)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200.config import ExperimentConfig  # noqa: E402
from paper_2503_15448_b200.experiment import build_world  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, GlobalState  # noqa: E402

cfg = dict(bench.C5_SHARE, rounds=6)
world, init = build_world(ExperimentConfig.from_dict(cfg), precision="bf16")
eng = FederationEngine(world)
st = eng.run_sync_round(GlobalState(round=0, w_g=init))
torch.cuda.synchronize()
for rep in range(4):
    eng.trace = []
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    a.record()
    h0 = time.perf_counter()
    eng._mark("start")
    st = eng.run_sync_round(st)
    eng._mark("end")
    torch.cuda.synchronize()
    print(f"--- round {st.round - 1}")
    for label, h, ev in eng.trace:
        print(f"{label:40s} host {(h - h0) * 1e3:8.2f} ms   device {a.elapsed_time(ev):8.2f} ms")
