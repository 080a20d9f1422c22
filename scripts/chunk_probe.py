"""e2e rounds/s of C4 for several upload chunk sizes (diagnostic):
server.UPLOAD_CHUNK_MB set before the world's host pack is built."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import server as S  # noqa: E402

for mb in [float(a) for a in sys.argv[1:]] or [8.0, 4.0, 2.0, 16.0]:
    S.UPLOAD_CHUNK_MB = mb
    world, init = bench.build_c4_world(precision="bf16")
    m = bench.measure_rounds(world, init, None, 5, 3, 0)
    vals = [bench.measure_e2e(world, m["engine"], m["state"], 10, m["barrier"])[0] for _ in range(3)]
    print(f"chunk {mb:5.1f} MB: value {1000.0 / m['ms_per_round']:.1f}  e2e {sorted(vals)}", flush=True)
    del world, m
    torch.cuda.empty_cache()
