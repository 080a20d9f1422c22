"""C4 bf16 round time with K6 fused into the trainer vs the separate pass (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import server as S  # noqa: E402

world, init = bench.build_c4_world(precision="bf16")
for rep in range(3):
    for mode in (False, True):
        S._FUSED_ALIGN = mode
        m = bench.measure_rounds(world, init, None, 20, 5, 0)
        k = m["kernels"]
        print(f"fused={mode}: {m['ms_per_round']:.3f} ms/round ({1000 / m['ms_per_round']:.1f} rounds/s) "
              f"train {k['train']['mean_ms']:.3f} agg {k['aggregate']['mean_ms']:.3f} "
              f"align {k.get('align', {}).get('mean_ms', 0):.3f}", flush=True)
