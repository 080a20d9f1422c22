"""Why the C5-share rounds are slower inside the full bench (diagnostic):
the bench's earlier stages in order, the C5-share measurement after each,
with the device memory picture."""
import gc
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def mem(tag):
    free, tot = torch.cuda.mem_get_info()
    print(f"{tag:28s} free {free / 2**30:6.1f} GiB  reserved {torch.cuda.memory_reserved() / 2**30:6.1f} GiB  "
          f"allocated {torch.cuda.memory_allocated() / 2**30:6.1f} GiB", flush=True)


def c5(tag):
    d = bench.measure_c5_share("bf16")
    print(f"  C5 after {tag}: {d['ms_per_round']:.1f} ms/round (train {d['train_ms']:.1f})", flush=True)
    mem("  after C5")


gc.collect()
gc.freeze()
mem("start")
world, initial = bench.build_c4_world(precision="bf16")
m = bench.measure_rounds(world, initial, None, 5, 3, 0)
bench.measure_e2e(world, m["engine"], m["state"], 2, m["barrier"])
mem("C4 bf16 + e2e")
c5("C4")
w64, i64 = bench.build_c4_world(precision="fp64")
p = bench.measure_rounds(w64, i64, None, 3, 3, 0)
bench.measure_e2e(w64, p["engine"], p["state"], 2, p["barrier"])
mem("fp64")
c5("fp64")
bench.measure_quality("bf16")
bench.measure_quality("fp64")
mem("quality")
c5("quality")
bench.hbm_microbench()
bench.hbm_microbench(52225, 1024, 400)
mem("micro")
c5("micro")
bench.measure_async("bf16")
mem("async")
c5("async")
