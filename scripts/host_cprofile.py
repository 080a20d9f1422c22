"""cProfile of the host side of C4 bf16 sync rounds (diagnostic)."""
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
pr.enable()
for _ in range(20):
    st = eng.run_sync_round(st)
torch.cuda.synchronize()
pr.disable()
ps = pstats.Stats(pr)
ps.sort_stats("tottime").print_stats(25)
ps.sort_stats("cumulative").print_callees("run_trainer")
ps.sort_stats("cumulative").print_callees("_prefetch_plan")
ps.sort_stats("cumulative").print_callees("_capture_global")
ps.sort_stats("cumulative").print_callees("keep")
ps.sort_stats("cumulative").print_callees("_emit_report")
