import os, sys, time, gc
import torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2503_15448_b200.server import FederationEngine, GlobalState
world, init = bench.build_c4_world(precision="bf16")
eng = FederationEngine(world)
st = GlobalState(round=0, w_g=init)
for _ in range(3):
    st = eng.run_sync_round(st)
torch.cuda.synchronize()
gcs = []
gc.callbacks.append(lambda phase, info: gcs.append((phase, info.get("generation"), time.perf_counter())))
ms = []
for i in range(30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    st = eng.run_sync_round(st)
    b.record()
    torch.cuda.synchronize()
    ms.append((round(a.elapsed_time(b), 2), round(1e3 * (time.perf_counter() - t0), 2)))
print(ms)
print("gc events", [(p, g) for p, g, _ in gcs][:20], len(gcs))
