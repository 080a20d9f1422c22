"""C4 async run times in a process holding a large heap (as bench.py does), to
expose host pauses (diagnostic; FS_ASYNC_PROF=1 prints per-phase host times)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

big = [bench.build_c4_world(precision="bf16"), bench.build_c4_world(precision="fp64")]
print(bench.measure_async("bf16", reps=int(os.environ.get("REPS", "8")))["run_s"], flush=True)
