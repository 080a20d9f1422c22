"""bf16 wide trainer vs fp32 emulation over seeds (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gpu_bf16 import _one_step  # noqa: E402

for dims, rows, dp in [((42, 1024, 1024, 1024, 1024, 1), 21, 0.0), ((42, 1024, 1024, 1024, 1024, 1), 64, 0.0),
                       ((42, 256, 128, 64, 1), 21, 0.0)]:
    rels = []
    for seed in range(1, 9):
        w0, got, want = _one_step(dims, rows, dp, seed=seed)
        rels.append(((got - want).norm() / (want - w0).norm()).item())
    print(dims, rows, dp, " ".join(f"{r:.1e}" for r in rels))
