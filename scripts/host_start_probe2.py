"""Host time from the start of a C4 bf16 sync round to its trainer launch
(diagnostic): cProfile callees of the calls made before the launch."""
import cProfile
import os
import pstats
import sys

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
pr = cProfile.Profile()
for _ in range(40):
    torch.cuda.synchronize()
    pr.enable()
    st = eng.run_sync_round(st)
    pr.disable()
torch.cuda.synchronize()
ps = pstats.Stats(pr)
ps.sort_stats("cumulative").print_callees("_run_sync_round_fast")
ps.sort_stats("cumulative").print_callees("run_trainer")
ps.sort_stats("cumulative").print_callees("run_sync_round")
ps.sort_stats("cumulative").print_callees("device_params")
