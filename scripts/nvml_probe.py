"""Which NVML query disturbs the GPU timeline? (diagnostic)"""
import os, sys, threading, time
import numpy as np
import torch
import pynvml as nv
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa
from paper_2503_15448_b200.server import FederationEngine, GlobalState

world, init = bench.build_c4_world(precision="bf16")
eng = FederationEngine(world)
st = GlobalState(round=0, w_g=init)
for _ in range(3):
    st = eng.run_sync_round(st)
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
fns = {"none": None, "clock": lambda: nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
       "maxclock": lambda: nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
       "reasons": lambda: nv.nvmlDeviceGetCurrentClocksEventReasons(h)}
for name, f in fns.items():
    stop = threading.Event()
    calls = [0]
    def loop():
        while not stop.is_set():
            if f:
                t = time.perf_counter(); f(); calls[0] += 1
            stop.wait(0.02)
    th = threading.Thread(target=loop, daemon=True); th.start()
    ms = []
    for _ in range(40):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); st = eng.run_sync_round(st); b.record(); torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    stop.set(); th.join()
    ms = np.array(ms)
    print(f"{name:9s} calls {calls[0]:4d} median {np.median(ms):.2f} max {ms.max():.2f} n>4ms {(ms > 4).sum()}")
