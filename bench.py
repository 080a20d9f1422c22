"""Benchmark: FL rounds/sec and client-updates/sec at 1024 UNSW-shaped clients.

Workload (BASELINE.json configs[3], SURVEY.md §8d "C4"): synthetic
UNSW-NB15-shaped data (219,176 rows x 42 features, 30 % anomalies, Dirichlet
alpha=0.5 over 1024 clients), the 42-256-128-64-1 MLP with dropout 0.3,
E=5 local epochs, capacity-driven batch sizes (dynamic 64..1024),
gradient-sign (delta_sign) selection at theta=0.65, FedAvg, per-round
evaluation on the 43,835-row test split. One bench "step" is one
synchronous FL round over all 1024 clients (training, selection,
aggregation, evaluation, event-log bookkeeping). Default precision is the
bf16 tensor-core mode (fp32 master weights); the fp64 parity mode (event
log bit-identical to the reference's) is measured in the same run and
reported under "fp64_parity".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--gpus N outside torchrun re-launches itself as N ranks (torch.distributed.run,
127.0.0.1). --impl reference times the REFERENCE package itself
(oracle/_ref/pkg, built by oracle/build_ref.sh): K consecutive full C4 rounds
of its own FederationEngine.run_sync_round, its client fan-out on forked
workers over every host core. The b200 arm's cpu_baseline is the same
package on one core, one full round. Prints ONE JSON line (rank 0); see
DESIGN.md §8 for every field.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

# CPU legs pin BLAS to one thread per process: the reference path is GIL- and
# per-call-overhead-bound (8 BLAS threads gave no speed-up);
# the reference arm gets every core through forked worker processes instead.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C4_SYNC = {
    "num_clients": 1024, "rounds": 100, "epochs": 5, "mode": "sync_filtered",
    "selection_mode": "delta_sign", "theta": 0.65, "seed": 1,
    "dataset": {"kind": "synthetic", "n": 219176, "d": 42, "anomaly_frac": 0.3, "separation": 4.0,
                "test_frac": 0.2},
    "model": {"hidden_dims": [256, 128, 64], "dropout_rate": 0.3},
    "batch": {"policy": "dynamic", "b_ref": 64, "b_min": 64, "b_max": 1024},
    "profiles": {"speed": {"distribution": "loguniform", "low": 20.0, "high": 200.0},
                 "capacity": {"distribution": "loguniform", "low": 0.25, "high": 4.0},
                 "up_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5},
                 "down_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5}},
    "lr": 0.05, "lr_decay": 0.9,
}
METRIC = "FL rounds/sec (1024 UNSW-shaped clients, C4 sync_filtered)"
C4_WORKLOAD = ("C4 sync_filtered: 1024 UNSW-shaped clients (175,341 train rows, d=42), MLP 42-256-128-64-1 "
               "dropout 0.3, E=5, dynamic batch 64..1024, delta_sign theta=0.65, FedAvg, eval on 43,835 rows")
N_DELTA = 1  # FS_ALIGN_DELTA_SIGN
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_NOMINAL_TFLOPS = 37.0  # B200 FP64 (CUDA-core and DMMA) nominal; no measured fp64 peak exists


def build_c4_world(num_clients: int = 1024, precision: str = "fp64"):
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world

    cfg = dict(C4_SYNC)
    cfg["num_clients"] = num_clients
    return build_world(ExperimentConfig.from_dict(cfg), precision=precision)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks + throttle reasons, sampled through NVML between the timed
    rounds of the timed region (`sample()` after each round's barrier).

    NVML clock/throttle queries stall the GPU for milliseconds (measured:
    scripts/nvml_probe.py), so a background sampler would land those stalls
    inside the rounds it is meant to observe; sampled between rounds, the
    clocks still reflect the load (they do not relax within microseconds)."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple] = []  # (sm_mhz, max_mhz, reasons bitmask)
        self._nv = self._h = None
        self._smi = None

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self._nv, self._h = nv, nv.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:
            self._smi = _SmiSampler(self.index).__enter__()
        self.sample()
        return self

    def sample(self) -> None:
        if self._nv is None:
            return
        nv, h = self._nv, self._h
        try:
            self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                 nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
                                 nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
        except Exception:
            pass

    def __exit__(self, *exc):
        if self._smi is not None:
            self._smi.__exit__(*exc)
            self.samples = self._smi.samples()
        return False

    def summary(self) -> dict:
        sm = [x[0] for x in self.samples]
        mx = [x[1] for x in self.samples]
        reasons = sorted({name for _, _, bits in self.samples for name, bit in self.REASONS if bits & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm), "how": "NVML, between timed rounds"}


class _SmiSampler:
    """nvidia-smi -lms fallback of ClockSampler."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=lambda: self.lines.extend(ln.strip() for ln in self.proc.stdout),
                             daemon=True).start()
            t_end = time.time() + 3.0
            while not self.lines and time.time() < t_end:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def samples(self) -> list[tuple]:
        out = []
        bits = [0x8, 0x40, 0x20, 0x4]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                mask = sum(b for b, v in zip(bits, parts[2:]) if v.lower() == "active")
                out.append((float(parts[0]), float(parts[1]), mask))
            except ValueError:
                continue
        return out


# ------------------------------------------------------------------ CPU sides
def reference_engine(workers: int):
    """The REFERENCE package (oracle/_ref/pkg: the shipped fedsim with its
    compiled Cython backend, built by oracle/build_ref.sh) on the C4 config:
    its own build_world, FederationEngine and run_sync_round. With workers > 1
    the reference's client fan-out (server.py:412-415, a GIL-bound thread
    pool) runs in forked processes instead (oracle/ref_pool.py)."""
    from oracle.ref_pool import patch_server_pool, use_reference

    use_reference("compiled")
    import fedsim.server
    from fedsim.config import ExperimentConfig
    from fedsim.experiment import build_world
    from fedsim.server import FederationEngine, GlobalState

    if workers > 1:
        patch_server_pool(fedsim.server)
    world, initial = build_world(ExperimentConfig.from_dict(dict(C4_SYNC)), workers=workers)
    return FederationEngine(world), GlobalState(round=0, w_g=initial)


def time_reference_rounds(workers: int, warmup: int, steps: int):
    """Wall-clock seconds of `steps` consecutive full C4 sync rounds of the
    reference (after `warmup` rounds; round 0 has no delta_sign scoring, so
    warmup >= 1 puts only scored rounds in the timed region)."""
    eng, state = reference_engine(workers)
    for _ in range(warmup):
        state = eng.run_sync_round(state)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        state = eng.run_sync_round(state)
        times.append(time.perf_counter() - t0)
    rep = eng.reports[-1]
    return times, {"round": state.round, "accuracy": rep.accuracy, "auc": rep.auc}


def run_reference(args, rank: int, world_size: int) -> None:
    if rank != 0:
        return
    procs = args.ref_procs if args.ref_procs > 0 else (os.cpu_count() or 1)
    times, quality = time_reference_rounds(procs, max(1, args.warmup), args.steps)
    sec = float(np.mean(times))
    value = 1.0 / sec
    sample = (f"{args.steps} consecutive full C4 sync rounds (1024 clients, after {max(1, args.warmup)} warm-up "
              f"rounds) of the reference package's own FederationEngine.run_sync_round, Cython backend, "
              f"1 BLAS thread per process; client fan-out over {procs} forked worker processes (the "
              f"reference's thread pool, server.py:412-415, is GIL-bound)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rounds/s", "n_gpus": world_size,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": C4_WORKLOAD},
        "cpu_baseline": {"value": value, "unit": "rounds/s", "cores": procs, "kind": "reference",
                         "sample": sample, "host_cores": os.cpu_count()},
        "e2e": {"value": value, "unit": "rounds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "client_updates_per_s": value * 1024,
        "round_s": [round(t, 3) for t in times],
        "quality": quality,
    }
    print(json.dumps(line), flush=True)


def reference_cpu_baseline():
    """cpu_baseline of the b200 arm: the reference package on ONE core (its
    default workers=1), one full C4 sync round (round 0: all 1024 clients
    train, FedAvg, evaluation; ~20 s of CPU work)."""
    eng, state = reference_engine(1)
    t0 = time.perf_counter()
    eng.run_sync_round(state)
    sec = time.perf_counter() - t0
    return {"value": 1.0 / sec, "unit": "rounds/s", "cores": 1, "kind": "reference",
            "sample": "one full C4 sync round (round 0: 1024 clients train 5 epochs, FedAvg, evaluation; "
                      "delta_sign scoring starts in round 1) of the reference package (oracle/_ref/pkg, "
                      "Cython backend, workers=1, 1 BLAS thread)", "seconds": sec}


# ------------------------------------------------------------------ GPU arm
def flush_l2(buf):
    buf.zero_()


def measure_rounds(world, initial, comm, steps: int, warmup: int, device_index: int):
    """Time `steps` sync rounds (after `warmup`) with CUDA events on the launching
    stream, L2 flushed between rounds, max over ranks. Returns a dict."""
    import torch

    from paper_2503_15448_b200 import device as D
    from paper_2503_15448_b200.server import FederationEngine, GlobalState

    rt = D.Runtime.get()
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device=rt.device)
    dist = None
    if comm is not None:
        import torch.distributed as dist

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    eng = FederationEngine(world, comm=comm)
    state = GlobalState(round=0, w_g=initial)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        state = eng.run_sync_round(state)
    barrier()
    D.Runtime.timer = D.KernelTimer()
    calls0 = D.Runtime.abi_calls
    trainings0 = eng.trainings
    round_ms = []
    import gc

    gc.disable()  # no collector pauses inside the timed rounds (re-enabled below)
    with ClockSampler(device_index) as clocks:
        for _ in range(steps):
            flush_l2(l2_flush)
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            state = eng.run_sync_round(state)
            b.record(stream)
            barrier()
            clocks.sample()
            round_ms.append(a.elapsed_time(b))
    gc.enable()
    timer, D.Runtime.timer = D.Runtime.timer, None
    total_ms = float(np.sum(round_ms))
    if dist is not None:
        t = torch.tensor([total_ms], device=rt.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    return {"engine": eng, "state": state, "ms_per_round": total_ms / steps, "round_ms": round_ms,
            "kernels": timer.summary(), "abi_calls": D.Runtime.abi_calls - calls0,
            "trainings": eng.trainings - trainings0, "clocks": clocks.summary(), "barrier": barrier}


def measure_e2e(world, eng, state, reps: int, barrier, warmup: int = 3):
    """Same metric through the public API with HOST inputs: every step uploads
    the world's shards and test set from page-locked host memory and reads w_g
    back; `warmup` untimed steps of the same kind first."""
    import torch

    stream = torch.cuda.current_stream()
    world.host_pack()  # page-locked host copies prepared once, outside the timed region
    e2e_ms = []
    h2d = d2h = 0
    for i in range(reps + warmup):
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dev = world.upload()  # this step's inputs: host -> HBM
        state = eng.run_sync_round(state)
        host_w = state.w_g.values
        b.record(stream)
        barrier()
        if i >= warmup:
            e2e_ms.append(a.elapsed_time(b))
        h2d = dev.h2d_bytes
        d2h = host_w.nbytes + world.num_clients * 8 * 2
    return 1000.0 / float(np.mean(e2e_ms)), int(h2d), int(d2h)


NCU_TRAFFIC_FILE = "profiles/r2_ncu_train_kernel.json"
NCU_TRAFFIC_SOURCE = f"{NCU_TRAFFIC_FILE} (dram read+write bytes, one ncu --set full launch)"


def _ncu_traffic():
    """dram__bytes_read+write of the trainer from the committed ncu capture (per launch)."""
    f = os.path.join(ROOT, NCU_TRAFFIC_FILE)
    try:
        return json.load(open(f))["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def hbm_microbench(M: int = 3193857, n_clients: int = 256, n_agg: int | None = None, reps: int = 10):
    """K6/K7 standalone (default: the C5 WIDE-MLP row length), float32 rows,
    `n_agg` of the rows aggregated: achieved GB/s. Arguments are staged on the
    device first; `reps` back-to-back launches are timed between two events."""
    import torch

    from paper_2503_15448_b200 import device as D

    rt = D.Runtime.get()
    ld = (M + 31) // 32 * 32
    W = torch.randn(n_clients, ld, device=rt.device, dtype=torch.float32)[:, :M]
    wg = torch.randn(M, device=rt.device, dtype=torch.float32)
    wp = torch.randn(M, device=rt.device, dtype=torch.float32)
    ptr_c = W.data_ptr() + np.arange(n_clients, dtype=np.uint64) * np.uint64(ld * 4)
    k = n_agg or n_clients
    d_all = rt.h2d(ptr_c.view(np.int64))
    d_agg = rt.h2d(ptr_c[:k].view(np.int64))
    counts = torch.empty(n_clients, dtype=torch.int64, device=rt.device)
    res = torch.empty(M, dtype=torch.float32, device=rt.device)
    d_job = rt.h2d(np.array([0, k, res.data_ptr()], dtype=np.uint64).view(np.int64))  # job_off {0, k}, job_out
    d_sorted = torch.empty(k, dtype=torch.int64, device=rt.device)
    ws = rt.scratch("agg_rowsplit_bench", rt.lib.fs_aggregate_rowsplit_workspace_bytes(M))
    stream = torch.cuda.current_stream()
    launch = {
        "align": (lambda: rt.call(rt.lib.fs_sign_align_shared(d_all.data_ptr(), wg.data_ptr(), wp.data_ptr(),
                                                              n_clients, M, N_DELTA, 4, counts.data_ptr(),
                                                              rt.stream), "align"),
                  4.0 * M * (n_clients + 2)),
        "aggregate": (lambda: rt.call(rt.lib.fs_aggregate_f32(d_agg.data_ptr(), k, M, res.data_ptr(), rt.stream),
                                      "agg"), 4.0 * M * (k + 1)),
        # bf16 sync rounds' FedAvg (row-split, canonical order + 16 row groups)
        "aggregate_rowsplit": (lambda: rt.call(rt.lib.fs_aggregate_rowsplit_f32(
            d_agg.data_ptr(), d_job.data_ptr(), k, M, d_sorted.data_ptr(), d_job.data_ptr() + 16, ws.data_ptr(),
            ws.numel(), rt.stream), "agg_split"), 4.0 * M * (k + 1)),
    }
    flush = torch.zeros(64 << 20, dtype=torch.float32, device=rt.device)
    out = {}
    for name, (fn, nbytes) in launch.items():
        fn()
        torch.cuda.synchronize()
        evs = []
        for _ in range(reps):
            # reading 256 MiB leaves L2 cold but clean (a write-flush would leave
            # dirty lines whose write-back lands in the timed kernel); the spin
            # keeps the GPU busy while the host queues the launch, so the
            # events bracket the kernel alone
            flush.sum()
            torch.cuda._sleep(400_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
        out[name] = {"ms": ms, "bytes": nbytes, "achieved_gbs": nbytes / ms / 1e6, "M": M,
                     "rows": n_clients if name == "align" else k,
                     "how": f"median of {reps} launches, each queued behind a 256 MiB read (cold, clean L2)"}
    return out


def measure_async(precision: str, windows: int = 2, reps: int = 5):
    """C4 `async_filtered` (the reference's buffered asynchronous engine: C++
    event loop driving the device executor, deferred batched training): windows
    of 1024 applied updates per second. One untimed warm-up run first (module
    load, memory pools), then `reps` timed runs (median reported: single runs
    vary 0.14-0.6 s with host scheduling), CUDA events on the launching stream."""
    import torch

    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world
    from paper_2503_15448_b200.server import FederationEngine

    cfg = dict(C4_SYNC)
    cfg.update({"mode": "async_filtered", "rounds": windows})
    world, init = build_world(ExperimentConfig.from_dict(cfg), precision=precision)
    world.device_state()
    for _ in range(2):  # warm-up (module load, memory arena, pools)
        FederationEngine(world).run(init)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    runs = []
    for _ in range(reps):
        eng = FederationEngine(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.run(init)
        b.record(stream)
        torch.cuda.synchronize()
        runs.append(a.elapsed_time(b) / 1e3)
    sec = float(np.median(runs))
    return {"value": windows / sec, "unit": "rounds/s (windows of 1024 applied updates)",
            "run_s": runs, "statistic": f"median of {reps} full runs (each {windows} windows)",
            "client_updates_per_s": eng.trainings / sec, "trainings": eng.trainings,
            "device_batches": eng.device_batches, "events": len(eng.timeline.log), "windows": windows,
            "precision": precision, "gpu_launches": getattr(eng, "async_launches", None),
            "host_s": dict(zip(("prep", "wait", "post"), getattr(eng, "async_host_s", (None,) * 3))),
            "engine": "C++ event loop + C++ device executor (server._ASYNC_ENGINE = \"device\")",
            "digest": eng.timeline.digest()}


C5_SHARE = {
    "num_clients": 1024, "rounds": 3, "epochs": 5, "mode": "sync_filtered", "selection_mode": "delta_sign",
    "theta": 0.65, "seed": 1,
    "dataset": {"kind": "synthetic", "n": 219176 // 8, "d": 42, "anomaly_frac": 0.3, "separation": 4.0,
                "test_frac": 0.2},
    "partition": {"alpha": 5.0},
    "model": {"hidden_dims": [1024, 1024, 1024, 1024], "dropout_rate": 0.3},
    "batch": {"policy": "fixed", "size": 64},
    "profiles": C4_SYNC["profiles"],
}


def measure_small_configs(precision: str):
    """BASELINE configs[0] (C1: 10 UNSW clients, sync_baseline, b = 64),
    configs[1] (C2: 100 UNSW clients, async_filtered, dynamic batch,
    delta_sign) and configs[2] (C3: 256 ROAD-shaped CAN-window clients, d = 64,
    sync_filtered + async_filtered, b = 64): throughput of full runs after a
    warm-up run, CUDA events on the launching stream."""
    import torch

    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world
    from paper_2503_15448_b200.server import FederationEngine

    base = {"epochs": 5, "theta": 0.65, "seed": 1, "selection_mode": "delta_sign", "profiles": C4_SYNC["profiles"],
            "model": {"hidden_dims": [256, 128, 64], "dropout_rate": 0.3}}
    cfgs = {
        # BASELINE configs[0] (the reference's CPU run): 10 clients, 5 sync_baseline
        # rounds, b = 64; a 55k-row client's 4.3k sequential steps bound each round
        "c1_sync": dict(base, num_clients=10, rounds=5, mode="sync_baseline", selection_mode="weight_sign",
                        dataset=C4_SYNC["dataset"], batch={"policy": "fixed", "size": 64}),
        "c2_async": dict(base, num_clients=100, rounds=5, mode="async_filtered",
                         dataset=C4_SYNC["dataset"], batch=C4_SYNC["batch"]),
        "c3_sync": dict(base, num_clients=256, rounds=5, mode="sync_filtered", batch={"policy": "fixed", "size": 64},
                        dataset={"kind": "synthetic", "d": 64, "samples_per_client": 256, "anomaly_frac": 0.1,
                                 "separation": 2.0, "test_frac": 0.2}),
    }
    cfgs["c3_async"] = dict(cfgs["c3_sync"], mode="async_filtered")
    out = {}
    for name, cfg in cfgs.items():
        world, init = build_world(ExperimentConfig.from_dict(cfg), precision=precision)
        world.device_state()
        for _ in range(2):  # warm-up (first-run allocations and module state)
            FederationEngine(world).run(init)
        torch.cuda.synchronize()
        secs = []
        for _ in range(3):  # median of three whole runs (single runs vary with host scheduling)
            eng = FederationEngine(world)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            eng.run(init)
            b.record()
            torch.cuda.synchronize()
            secs.append(a.elapsed_time(b) / 1e3)
        sec = float(np.median(secs))
        out[name] = {"clients": cfg["num_clients"], "rounds": cfg["rounds"], "rounds_per_s": cfg["rounds"] / sec,
                     "client_updates_per_s": eng.trainings / sec, "trainings": eng.trainings,
                     "run_s": secs, "statistic": "median of 3 whole runs after 2 warm-up runs",
                     "digest": eng.timeline.digest()}
    return out


def measure_c5_share(precision: str, rounds: int = 5):
    """BASELINE configs[4] (WIDE MLP 42-1024x4-1, 8192 clients over 8 GPUs):
    the 1024-client share one GPU owns, ~21 rows per client (data scaled 1/8),
    sync_filtered rounds after one warm-up round, each timed with CUDA events;
    the median round is reported (all rounds listed)."""
    import torch

    from paper_2503_15448_b200 import device as D
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world
    from paper_2503_15448_b200.server import FederationEngine, GlobalState

    world, init = build_world(ExperimentConfig.from_dict(dict(C5_SHARE, rounds=rounds + 1)), precision=precision)
    eng = FederationEngine(world)
    st = eng.run_sync_round(GlobalState(round=0, w_g=init))
    torch.cuda.synchronize()
    D.Runtime.timer = D.KernelTimer()
    stream = torch.cuda.current_stream()
    import gc

    gc.disable()  # no collector pauses inside the timed rounds
    evs = []
    for _ in range(rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        st = eng.run_sync_round(st)
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    gc.enable()
    ks, D.Runtime.timer = D.Runtime.timer.summary(), None
    round_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.median(round_ms))
    tr = ks.get("train", {})
    return {"workload": "C5 share: 1024 clients, WIDE MLP 42-1024x4-1 dropout 0.3, b=64, E=5, alpha=5, delta_sign",
            "rounds_per_s": 1000.0 / ms, "client_updates_per_s": 1024 * 1000.0 / ms, "ms_per_round": ms,
            "round_ms": round_ms, "statistic": f"median of {rounds} rounds after one warm-up round",
            "train_ms": tr.get("mean_ms"),
            "train_tflops": (tr["work_per_launch"] / (tr["mean_ms"] * 1e-3) / 1e12) if tr else None,
            "trainer": "fs_train_wide.cu (factored bf16 tcgen05 trainer: shared start model + per-client history)"
            if precision == "bf16" else "fp64 parity trainer"}


def measure_c5_async_share(precision: str):
    """BASELINE configs[4] is async_filtered: the same 1024-client WIDE share
    through the async engine (C++ event loop + device executor driving the
    batched-GEMM trainer), one window; after a warm-up run on a 64-client world.
    Reported as client-updates/s (delta_sign rejects most WIDE updates, so the
    run ends at the reference's cycle budget before the window fills)."""
    import torch

    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world
    from paper_2503_15448_b200.server import FederationEngine

    warm = dict(C5_SHARE, mode="async_filtered", rounds=1, num_clients=64)
    warm["dataset"] = dict(C5_SHARE["dataset"], n=219176 * 64 // 8192)
    w, i = build_world(ExperimentConfig.from_dict(warm), precision=precision)
    FederationEngine(w).run(i)
    world, init = build_world(ExperimentConfig.from_dict(dict(C5_SHARE, mode="async_filtered", rounds=1)),
                              precision=precision)
    world.device_state()
    torch.cuda.synchronize()
    eng = FederationEngine(world)
    stream = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    eng.run(init)
    b.record(stream)
    torch.cuda.synchronize()
    sec = a.elapsed_time(b) / 1e3
    return {"workload": "C5 share, async_filtered: 1024 clients, WIDE MLP, 1 window",
            "client_updates_per_s": eng.trainings / sec, "trainings": eng.trainings, "seconds": sec,
            "windows_completed": len(eng.reports), "device_batches": eng.device_batches,
            "digest": eng.timeline.digest()}


def reference_quality(rounds: int = 5):
    """The reference's own per-round accuracy/AUC on C4 (committed fixture
    tests/golden/configs.json, recorded from the reference package by
    tests/golden/make_golden_configs.py)."""
    f = os.path.join(ROOT, "tests", "golden", "configs.json")
    try:
        rep = json.load(open(f))["c4_sync"]["reports"]
    except (OSError, KeyError, ValueError):
        return None
    return {"round": rounds - 1, "accuracy": rep[rounds - 1]["accuracy"], "auc": rep[rounds - 1]["auc"],
            "source": "reference package, tests/golden/configs.json (c4_sync)"}


def measure_quality(precision: str, rounds: int = 5):
    """Accuracy/AUC of the global model after `rounds` C4 rounds from the
    initial model (the bench's own world, this precision)."""
    from paper_2503_15448_b200.server import FederationEngine, GlobalState

    world, initial = build_c4_world(precision=precision)
    eng = FederationEngine(world)
    st = GlobalState(round=0, w_g=initial)
    for _ in range(rounds):
        st = eng.run_sync_round(st)
    rep = eng.reports[-1]
    return {"round": rounds - 1, "accuracy": rep.accuracy, "auc": rep.auc,
            "accepted": [r.accepted for r in eng.reports]}


def run_b200(args, rank: int, world_size: int) -> None:
    import gc

    import torch

    from paper_2503_15448_b200.parallel import ShardComm

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % max(torch.cuda.device_count(), 1))
    comm = ShardComm.from_env()
    gc.collect()
    gc.freeze()  # the worlds built below outlive the bench: keep them out of the collector's scans
    world, initial = build_c4_world(precision=args.precision)
    m = measure_rounds(world, initial, comm, args.steps, args.warmup, local)
    value = 1000.0 / m["ms_per_round"]
    e2e_value, h2d, d2h = measure_e2e(world, m["engine"], m["state"], max(5, args.steps // 2), m["barrier"],
                                      warmup=max(3, args.warmup))
    parity = None
    if not args.no_parity:
        w64, i64 = build_c4_world(precision="fp64")
        p = measure_rounds(w64, i64, comm, 3, 3, local)
        e64, h64, d64 = measure_e2e(w64, p["engine"], p["state"], 2, p["barrier"])
        parity = {"value": 1000.0 / p["ms_per_round"], "unit": "rounds/s", "ms_per_step": p["ms_per_round"],
                  "train_kernel_ms": p["kernels"].get("train", {}).get("mean_ms"),
                  "e2e": {"value": e64, "unit": "rounds/s", "h2d_bytes_per_step": h64, "d2h_bytes_per_step": d64},
                  "note": "fp64 parity mode: event log bit-identical to the reference (tests/test_gpu_parity.py)"}
    if rank != 0:
        if comm is not None:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    quality = None
    if world_size == 1 and not args.no_quality:
        quality = {"bf16": measure_quality("bf16"), "fp64": measure_quality("fp64"),
                   "reference": reference_quality(),
                   "note": "accuracy/AUC on the 43,835-row test split after 5 C4 rounds from the same initial "
                           "model; fp64 equals the reference exactly, bf16 is tolerance-matched"}
    ksum = m["kernels"]
    peaks = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
    tr = ksum.get("train", {})
    achieved = tr["work_per_launch"] / (tr["mean_ms"] * 1e-3) / 1e12 if tr else None
    if args.precision == "bf16":
        peak, src = peaks.get("bf16_tflops", 1590.0), ("MEASURED_PEAKS.json bf16_tflops (burst)" if peaks
                                                      else "B200_PROFILING.md fallback 1.59 PFLOP/s")
        roofline = {"kernel": "fs::bf16t::train_kernel (K5 unit-major, tcgen05/TMEM)", "bound": "tensor"}
    else:
        peak, src = FP64_NOMINAL_TFLOPS, "nominal B200 FP64 37 TFLOP/s (no measured fp64 peak)"
        roofline = {"kernel": "fs::f64::train_kernel (K5, fp64 parity)", "bound": "fp64"}
    roofline.update({"achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if achieved else None, "peak_source": src,
                     "traffic": _ncu_traffic() if args.precision == "bf16" else None,
                     "traffic_source": NCU_TRAFFIC_SOURCE,
                     "algorithmic_flops_per_launch": tr.get("work_per_launch"),
                     "share_of_round": tr.get("total_ms", 0.0) / (m["ms_per_round"] * args.steps) if tr else None})
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    kernels = {}
    for name in ("align", "aggregate"):
        if name in ksum:
            k = ksum[name]
            gbs = k["work_per_launch"] / (k["mean_ms"] * 1e-3) / 1e9
            kernels[name] = {"achieved_gbs": gbs, "frac_hbm": gbs / hbm_peak, "mean_ms": k["mean_ms"],
                             "bytes_per_launch": k["work_per_launch"]}
    c5 = c4_micro = None
    if not args.no_micro:
        c5 = hbm_microbench()
        c4_micro = hbm_microbench(52225, 1024, 400)
        for v in list(c5.values()) + list(c4_micro.values()):
            v["frac_hbm"] = v["achieved_gbs"] / hbm_peak
    async_c4 = None
    if world_size == 1 and not args.no_async:
        async_c4 = measure_async(args.precision)
    c5_share = small = None
    if world_size == 1 and not args.no_c5:
        c5_share = measure_c5_share(args.precision)
        c5_share["async"] = measure_c5_async_share(args.precision)
        small = measure_small_configs(args.precision)
    cpu = None
    if world_size == 1 and not args.no_cpu:
        try:
            cpu = reference_cpu_baseline()
        except ImportError as e:  # oracle/_ref not shipped with this snapshot
            cpu = {"value": None, "unit": "rounds/s", "cores": 1, "kind": "reference", "unavailable": str(e)}
    line = {
        "metric": METRIC, "value": value, "unit": "rounds/s", "n_gpus": world_size, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["ms_per_round"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16" if args.precision == "bf16" else "f64", "data": "synthetic",
        "config": {"workload": C4_WORKLOAD,
                   "precision": ("bf16 GEMM operands, fp32 accumulate/master weights (tolerance-matched)"
                                 if args.precision == "bf16" else "fp64 parity (digest-identical to reference)"),
                   "l2": "256 MiB buffer written between timed rounds (L2 flush)",
                   "parallelism": f"1024 clients sharded over {world_size} GPU(s), 1 NCCL all-reduce/round"},
        "client_updates_per_s": value * m["trainings"] / args.steps,
        "e2e": {"value": e2e_value, "unit": "rounds/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "note": "public World.upload + FederationEngine.run_sync_round: shards + test set copied from "
                        "page-locked host memory into HBM every step (bf16 mode: the trainer's bf16 row format, "
                        "converted once at world build), w_g read back"},
        "roofline": roofline,
        "hbm_kernels": {"c4_standalone": c4_micro, "c5_standalone": c5, "c4_in_round": kernels,
                        "note": "standalone: each launch timed alone behind a 256 MiB read (cold, clean L2); "
                                "in_round: CUDA events around the launch inside the timed rounds, where the "
                                "next round's K2/K3 prefetch shares the SMs (overlap by design)"},
        "fp64_parity": parity,
        "quality": quality,
        "async_c4": async_c4,
        "c5_share_1gpu": c5_share,
        "c2_c3_1gpu": small,
        "cpu_baseline": cpu,
        "gpu_launches": int(m["abi_calls"]),
        "gpu_launches_note": "kernel-launching C-ABI calls in the timed region (a CUB sort counts as one)",
        "clocks": m["clocks"],
        "kernel_ms": {k: v["mean_ms"] for k, v in ksum.items()},
        "round_ms": [round(x, 3) for x in m["round_ms"]],
    }
    print(json.dumps(line), flush=True)
    if comm is not None:
        import torch.distributed as dist

        dist.destroy_process_group()


def spawn_ranks(n: int) -> int:
    """`--gpus N` outside torchrun: relaunch this command as N ranks (one per
    GPU) under torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-procs", type=int, default=0, help="worker processes for the reference arm (0: all cores)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--precision", default="bf16", choices=["fp64", "bf16"])
    ap.add_argument("--no-parity", action="store_true", help="skip the fp64 parity-mode measurement")
    ap.add_argument("--no-quality", action="store_true", help="skip the 5-round accuracy/AUC check")
    ap.add_argument("--no-micro", action="store_true", help="skip the C5-shape HBM microbenchmark")
    ap.add_argument("--no-async", action="store_true", help="skip the C4 async-engine measurement")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5-share (WIDE MLP) measurement")
    args = ap.parse_args()
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank, world_size)
    else:
        run_b200(args, rank, world_size)


if __name__ == "__main__":
    main()
