"""Host-time breakdown of the end-to-end leg (device world rebuilt from host memory)."""
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
host = world.host_pack()
for k, v in (("x", host["shards"].x), ("y", host["shards"].y), ("tx", host["test_x"]), ("ty", host["test_y"])):
    print(k, v.dtype, tuple(v.shape), "pinned", v.is_pinned())
for _ in range(3):
    world._device = None
    st = eng.run_sync_round(st)
    _ = st.w_g.values
torch.cuda.synchronize()
for rep in range(4):
    world._device = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dx = host["shards"].x.to("cuda", non_blocking=True)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dev = world.device_state()
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    st = eng.run_sync_round(st)
    _ = st.w_g.values
    t5 = time.perf_counter()
    print(f"x.to {1e3*(t1-t0):.2f} ms (+sync {1e3*(t2-t1):.2f}); device_state {1e3*(t3-t2):.2f} (+sync {1e3*(t4-t3):.2f}); round {1e3*(t5-t4):.2f}")
    del dx
