"""Device timeline of C4 bf16 e2e rounds (World.upload + run_sync_round +
reading w_g back, as bench.py's e2e leg) via torch.profiler/CUPTI
(diagnostic; timings under the profiler are not bench values)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_15448_b200.server import FederationEngine, GlobalState  # noqa: E402

if os.environ.get("TRACE_C3"):  # the C3 world (256 ROAD clients, b = 64) instead of C4
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world

    cfg = {"epochs": 5, "theta": 0.65, "seed": 1, "selection_mode": "delta_sign", "profiles": bench.C4_SYNC["profiles"],
           "model": {"hidden_dims": [256, 128, 64], "dropout_rate": 0.3}, "num_clients": 256, "rounds": 100,
           "mode": "sync_filtered", "batch": {"policy": "fixed", "size": 64},
           "dataset": {"kind": "synthetic", "d": 64, "samples_per_client": 256, "anomaly_frac": 0.1,
                       "separation": 2.0, "test_frac": 0.2}}
    world, init = build_world(ExperimentConfig.from_dict(cfg), precision="bf16")
else:
    world, init = bench.build_c4_world(precision="bf16")
eng = FederationEngine(world)
state = GlobalState(round=0, w_g=init)
for _ in range(4):
    state = eng.run_sync_round(state)
torch.cuda.synchronize()
l2 = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        l2.add_(1)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("round")
        world.upload()
        state = eng.run_sync_round(state)
        _ = state.w_g.values
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
out = os.path.join("gpurun_out", "e2e_trace.json")
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
keep = []
for e in ev:
    if e.get("ph") != "X":
        continue
    cat = e.get("cat", "")
    if cat in ("kernel", "gpu_memcpy", "gpu_memset", "cuda_runtime", "cuda_driver"):
        keep.append({"cat": cat, "name": e["name"][:70], "ts": e["ts"], "dur": e["dur"],
                     "stream": e.get("args", {}).get("stream"), "tid": e.get("tid")})
keep.sort(key=lambda e: e["ts"])
json.dump(keep, open(os.path.join("gpurun_out", "e2e_trace_slim.json"), "w"))
print(len(keep), "events")
