"""Wall-clock phases of one device-mode async run (diagnostic)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200 import async_loop, server  # noqa: E402
from paper_2503_15448_b200.config import ExperimentConfig  # noqa: E402
from paper_2503_15448_b200.experiment import build_world  # noqa: E402

T = {}
orig_init, orig_attach, orig_run, orig_log, orig_close = (async_loop.AsyncLoop.__init__, async_loop.AsyncLoop.attach_device,
                                                          async_loop.AsyncLoop.run, async_loop.AsyncLoop.log_block,
                                                          async_loop.AsyncLoop.close)


def timed(name, fn):
    def w(*a, **k):
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            T[name] = T.get(name, 0.0) + time.perf_counter() - t
    return w


async_loop.AsyncLoop.__init__ = timed("loop init", orig_init)
async_loop.AsyncLoop.attach_device = timed("attach", orig_attach)
async_loop.AsyncLoop.run = timed("run", orig_run)
async_loop.AsyncLoop.log_block = timed("log_block", orig_log)
async_loop.AsyncLoop.close = timed("close", orig_close)
cfg = dict(bench.C4_SYNC)
cfg.update({"mode": "async_filtered", "rounds": 2})
world, init = build_world(ExperimentConfig.from_dict(cfg), precision="bf16")
world.device_state()
for rep in range(2):
    T.clear()
    torch.cuda.synchronize()
    eng = server.FederationEngine(world)
    t0 = time.perf_counter()
    eng.run(init)
    torch.cuda.synchronize()
    print(f"total {time.perf_counter() - t0:.3f}s", {k: round(v, 4) for k, v in T.items()}, eng.async_host_s)
