"""K6/K7 standalone HBM rates at the C4 and C5 row lengths (bench.hbm_microbench) (diagnostic)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for name, args in (("c4", (52225, 1024, 400)), ("c5", ())):
    r = bench.hbm_microbench(*args)
    print(name, json.dumps({k: round(v["achieved_gbs"]) for k, v in r.items()}), flush=True)
