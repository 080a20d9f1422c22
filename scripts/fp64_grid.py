"""fp64 parity-mode C4 round time vs trainer grid (diagnostic; FS_TRAIN_GRID read at import)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import device as D  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, GlobalState  # noqa: E402

world, init = bench.build_c4_world(precision="fp64")
eng = FederationEngine(world)
st = GlobalState(round=0, w_g=init)
st = eng.run_sync_round(st)
torch.cuda.synchronize()
D.Runtime.timer = D.KernelTimer()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    st = eng.run_sync_round(st)
b.record()
torch.cuda.synchronize()
print(f"grid {os.environ.get('FS_TRAIN_GRID', 'auto')}: {a.elapsed_time(b) / 3:.1f} ms/round, "
      f"train {D.Runtime.timer.summary()['train']['mean_ms']:.1f} ms")
