"""K6/K7 standalone at the C4 (UNSW MLP) and C5 (WIDE) row lengths (diagnostic)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for name, M, n, k in (("c4", 52225, 1024, 400), ("c4_all", 52225, 1024, 1024), ("c5", 3193857, 256, 256)):
    print(name, json.dumps(bench.hbm_microbench(M, n, k)))
