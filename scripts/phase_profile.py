"""Per-phase cycle breakdown of the bf16 trainer on one C4 round (diagnostic)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import _native as N  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, GlobalState  # noqa: E402

NAMES = {0: "gather", 1: "F0 mma", 2: "F1 mma", 3: "F2 mma", 5: "F0 epi", 6: "F1 epi", 7: "F2 epi+z",
         9: "head z/dz", 10: "head grads", 11: "D_L-1 + head upd", 12: "B0 mma", 13: "B1 mma", 14: "B2 mma",
         16: "B0 D-epi", 17: "B1 D-epi", 18: "B2 D-epi", 20: "B0 G-epi", 21: "B1 G-epi", 22: "B2 G-epi",
         24: "bias grads (last stage)", 25: "chunk end barrier", 26: "client setup: W0 + biases", 27: "client end sync", 28: "X tile stores", 29: "mask finish", 30: "client: write-back + claim", 31: "client setup: W1/W2"}
world, init = bench.build_c4_world(precision="bf16")
eng = FederationEngine(world)
st = GlobalState(round=0, w_g=init)
st = eng.run_sync_round(st)
lib = N.load()
prof = torch.zeros(32, dtype=torch.int64, device="cuda")
lib.fs_bf16_set_profile(prof.data_ptr())
st = eng.run_sync_round(st)
torch.cuda.synchronize()
lib.fs_bf16_set_profile(None)
p = prof.cpu().numpy().astype(float)
tot = p.sum()
for k in range(32):
    if p[k]:
        print(f"{k:2d} {NAMES.get(k, '?'):28s} {100 * p[k] / tot:6.2f}%  {p[k] / 148 / 1.9e3:9.1f} us/SM")
print("total cycles/SM", tot / 148)
