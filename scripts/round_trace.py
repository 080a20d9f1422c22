"""Host/device timeline of one C4 sync round (diagnostic)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, GlobalState  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
world, init = bench.build_c4_world(precision=prec)
eng = FederationEngine(world)
st = GlobalState(round=0, w_g=init)
for _ in range(3):
    st = eng.run_sync_round(st)
torch.cuda.synchronize()
E2E = os.environ.get("E2E") == "1"  # rebuild the device world from host memory each round
if E2E:
    world.host_pack()
for rep in range(2):
    eng.trace = []
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    if E2E:
        world._device = None
        world.device_state()
        eng._mark("device world rebuilt")
    st = eng.run_sync_round(st)
    if E2E:
        _ = st.w_g.values
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"round: host {1e3 * (t1 - t0):.2f} ms, device {e0.elapsed_time(e1):.2f} ms")
    for label, th, ev in eng.trace:
        print(f"  {label:36s} host +{1e3 * (th - t0):7.2f} ms   device-queue +{e0.elapsed_time(ev):7.2f} ms")
