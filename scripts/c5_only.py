"""C5 share sync + async measurement alone (diagnostic)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for _ in range(2):
    r = bench.measure_c5_share("bf16")
    print(json.dumps({k: r[k] for k in ("rounds_per_s", "ms_per_round", "train_ms")}), flush=True)
