"""Host microseconds from entering run_sync_round to the trainer's launch
call (diagnostic): wrapped functions record perf_counter stamps."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import device as D  # noqa: E402
from paper_2503_15448_b200 import server as S  # noqa: E402

stamps = []


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        stamps.append((name + ">", time.perf_counter()))
        r = f(*a, **k)
        stamps.append((name + "<", time.perf_counter()))
        return r
    setattr(mod, name, g)


for n in ("device_params", "top_k_mask", "score_denominator"):
    if hasattr(S, n):
        wrap(S, n)
for n in ("run_trainer", "_launch_trainer", "fused_align_supported"):
    wrap(D, n)
lib_call = D.Runtime.call


def call(self, rc, what):
    stamps.append(("call " + what, time.perf_counter()))
    return lib_call(self, rc, what)


D.Runtime.call = call
world, init = bench.build_c4_world(precision="bf16")
eng = S.FederationEngine(world)
st = S.GlobalState(round=0, w_g=init)
for _ in range(4):
    st = eng.run_sync_round(st)
torch.cuda.synchronize()
D.Runtime.timer = D.KernelTimer() if len(sys.argv) > 1 else None
rows = {}
for rep in range(20):
    torch.cuda.synchronize()
    stamps.clear()
    t0 = time.perf_counter()
    st = eng.run_sync_round(st)
    seen = {}
    for lab, t in stamps:
        if lab in seen:
            continue
        seen[lab] = 1
        rows.setdefault(lab, []).append((t - t0) * 1e6)
        if lab == "call fs_train_bf16":
            break
for lab, v in rows.items():
    print(f"{lab:40s} {np.median(v):8.1f} us")
