"""Per-round times over many C4 sync rounds; traces of the slow ones (diagnostic)."""
import gc
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, GlobalState  # noqa: E402

world, init = bench.build_c4_world(precision="bf16")
eng = FederationEngine(world)
st = GlobalState(round=0, w_g=init)
for _ in range(3):
    st = eng.run_sync_round(st)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
SAMPLER = None
if os.environ.get("NVML") == "1":
    SAMPLER = bench.ClockSampler(0).__enter__()
gc_events = []
gc.callbacks.append(lambda phase, info: gc_events.append((phase, info.get("generation"), time.perf_counter())))
times = []
for i in range(40):
    flush.zero_()
    torch.cuda.synchronize()
    eng.trace = []
    gc_events.clear()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    st = eng.run_sync_round(st)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    times.append(ms)
    if SAMPLER is not None:
        SAMPLER.sample()
    if ms > 3.5:
        print(f"round {i}: {ms:.2f} ms, gc {[(p, g, round(1e3 * (t - t0), 2)) for p, g, t in gc_events]}")
        for label, th, ev in eng.trace:
            print(f"   {label:36s} host +{1e3 * (th - t0):7.2f} ms   device +{a.elapsed_time(ev):7.2f} ms")
print("median", sorted(times)[len(times) // 2], "max", max(times), "n>3.5", sum(t > 3.5 for t in times))
