"""C5 share (WIDE MLP, 1024 clients) sync rounds alone (diagnostic; ncu target)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(reps):
    r = bench.measure_c5_share("bf16", rounds=1)
    print(json.dumps({k: r[k] for k in ("rounds_per_s", "ms_per_round", "train_ms", "train_tflops")}), flush=True)
