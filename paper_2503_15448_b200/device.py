"""Device runtime: resident shard store and the batched round-level operators.

The reference runs its round loop one client at a time (server.py:409-417
-> client.train_local -> backend.loss_and_grad per batch). Here the engines
hand a whole round (or a deferred batch of async trainings) to the GPU:

    train_requests   K1 seeds -> K2 shuffles -> K3 dropout bits -> K5 trainer
    align_requests   K6 sign-alignment counts (one launch for all clients)
    aggregate_rows   K9 sort keys -> host sort -> K7 ordered mean
    evaluate_global  K8 eval forward + accuracy/AUC counts

Only per-request metadata crosses the PCIe bus (one packed H2D per launch
group) plus the integer results the event log needs (aligned counts,
divergence flags). Parameters, shards, permutations and masks stay in HBM.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class _TimedLaunch:
    __slots__ = ("timer", "name", "work", "stream", "a", "b")

    def __init__(self, timer, name, work, stream):
        self.timer, self.name, self.work, self.stream = timer, name, work, stream

    def __enter__(self):
        self.a, self.b = self.timer._event(), self.timer._event()
        self.a.record(self.stream)
        return self

    def __exit__(self, *exc):
        self.b.record(self.stream)
        self.timer.events.setdefault(self.name, []).append((self.a, self.b, self.work))
        return False


class KernelTimer:
    """Optional CUDA-event brackets around the hot launches (bench/profiling).

    ``record(name, work)`` returns a context manager that records events on
    the launching stream; ``summary()`` reports mean duration per launch and
    the algorithmic work (FLOPs or bytes) each launch carried.
    """

    def __init__(self, prealloc: int = 512):
        self.events: dict[str, list] = {}
        self.launches = 0
        # CUDA events are created on their first record: a primed pool keeps
        # cudaEventCreate out of the launch path of the timed rounds
        self._pool = [torch.cuda.Event(enable_timing=True) for _ in range(prealloc)]
        for ev in self._pool:
            ev.record()

    def _event(self):
        return self._pool.pop() if self._pool else torch.cuda.Event(enable_timing=True)

    def record(self, name: str, work: float, stream) -> "_TimedLaunch":
        """Events around the launch; `ctx.work` may be set inside the block,
        after the launch, so the host never delays the kernel to count it."""
        return _TimedLaunch(self, name, work, stream)

    def summary(self) -> dict:
        out = {}
        for name, evs in self.events.items():
            ms = [a.elapsed_time(b) for a, b, _ in evs]
            work = [w for _, _, w in evs]
            out[name] = {"launches": len(evs), "mean_ms": float(np.mean(ms)), "total_ms": float(np.sum(ms)),
                         "work_per_launch": float(np.mean(work)), "work_total": float(np.sum(work))}
        return out


class Runtime:
    """Per-device state: stream handle and growable scratch buffers."""

    timer: KernelTimer | None = None   # set by bench.py to time hot launches
    abi_calls = 0                      # kernel-launching C-ABI calls issued

    _instances: dict[int, "Runtime"] = {}

    def __init__(self, index: int):
        self.lib = N.load(require_gpu=True)
        self.index = index
        self.device = torch.device("cuda", index)
        self._ws: dict[str, torch.Tensor] = {}
        self._streams: dict[str, torch.cuda.Stream] = {}

    def named_stream(self, role: str, high_priority: bool = False) -> torch.cuda.Stream:
        """A process-wide stream per role (engine main/side, uploads, checkpoint
        spills). Engines share them: every engine's work is ordered by stream
        order and events anyway, and the caching allocator reuses freed blocks
        only on the stream they were allocated on, so a fresh stream per engine
        turned each new engine's pooled buffers into cudaMalloc calls
        (device-synchronising; up to 0.3 s of a C3 run)."""
        st = self._streams.get(role)
        if st is None:
            prio = torch.cuda.Stream.priority_range()[1] if high_priority else 0
            st = self._streams[role] = torch.cuda.Stream(device=self.device, priority=prio)
        return st

    @classmethod
    def get(cls, index: int | None = None) -> "Runtime":
        N.load(require_gpu=True)
        if index is None:
            index = torch.cuda.current_device()
        rt = cls._instances.get(index)
        if rt is None:
            rt = cls(index)
            cls._instances[index] = rt
        return rt

    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def scratch(self, name: str, nbytes: int) -> torch.Tensor:
        """A cached uint8 device buffer of at least ``nbytes`` (stream-ordered reuse)."""
        nbytes = max(int(nbytes), 1)
        buf = self._ws.get(name)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 2 * (buf.numel() if buf is not None else 0)),
                              dtype=torch.uint8, device=self.device)
            self._ws[name] = buf
        return buf

    def h2d(self, arr: np.ndarray) -> torch.Tensor:
        """Pinned host copy -> device tensor (async on the current stream)."""
        src = torch.from_numpy(np.ascontiguousarray(arr))
        if src.numel() == 0:
            return torch.empty(0, dtype=src.dtype, device=self.device)
        return src.pin_memory().to(self.device, non_blocking=True)

    def call(self, rc: int, what: str) -> None:
        Runtime.abi_calls += 1
        N.check(rc, what)

    def timed(self, name: str, work: float):
        t = Runtime.timer
        if t is None:
            return _NULL_CTX
        return t.record(name, work, torch.cuda.current_stream(self.device))


class _Null:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


_NULL_CTX = _Null()


class Stage:
    """Page-locked host bump arena + device mirror for per-launch metadata.

    ``put`` packs a small array into the host arena and returns the device
    address it will have; ``commit`` issues ONE async copy of everything put
    since the last commit (instead of a pin_memory + copy per array). The
    caller ``reset``s the arena only after a host synchronisation that
    covers the previous copies (the async engine resets once per flush)."""

    def __init__(self, rt: "Runtime", nbytes: int = 1 << 20):
        self.rt = rt
        self._old: list = []
        self._alloc(nbytes)

    def _alloc(self, n: int) -> None:
        self.host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        self.hnp = self.host.numpy()
        self.dev = torch.empty(n, dtype=torch.uint8, device=self.rt.device)
        self.dbase = self.dev.data_ptr()
        self.off = self.done = 0

    def reset(self) -> None:
        self.off = self.done = 0
        self._old.clear()

    def put(self, arr: np.ndarray) -> int:
        b = np.ascontiguousarray(arr).reshape(-1).view(np.uint8)
        n = b.size
        start = (self.off + 15) & ~15
        if start + n > self.hnp.size:
            self.commit()
            self._old.append((self.host, self.dev))  # in flight: keep until reset
            self._alloc(max(2 * self.hnp.size, 2 * n))
            start = 0
        self.hnp[start:start + n] = b
        self.off = start + n
        return self.dbase + start

    def commit(self, stream=None) -> None:
        if self.off > self.done:
            s = stream if stream is not None else torch.cuda.current_stream(self.rt.device)
            with torch.cuda.stream(s):
                self.dev[self.done:self.off].copy_(self.host[self.done:self.off], non_blocking=True)
            self.done = self.off


def mlp_flops_per_sample(dims) -> int:
    """Algorithmic fwd+bwd FLOPs per sample: 4*sum f_l f_l+1 over
    all layers for forward + weight gradients, plus 2*sum over layers l>=1 for
    the input gradients of every layer but the first."""
    pairs = [a * b for a, b in zip(dims[:-1], dims[1:])]
    return 4 * sum(pairs) + 2 * sum(pairs[1:])


def dims_array(dims) -> tuple[ctypes.Array, int]:
    arr = (ctypes.c_int32 * len(dims))(*[int(d) for d in dims])
    return arr, len(dims)


# --------------------------------------------------------------------- shards
class HostPack:
    """Client shards packed once on the host ([rows x d] float64 + labels);
    with ``pin=True`` the buffers are page-locked, so uploads are plain async
    DMA copies (the bench's end-to-end leg re-uploads them every round)."""

    def __init__(self, features: list[np.ndarray], labels: list[np.ndarray], pin: bool = True, bf16: bool = False,
                 order: np.ndarray | None = None, chunk_bytes: int = 0):
        n_rows = np.array([f.shape[0] for f in features], dtype=np.int64)
        self.n_rows = n_rows.astype(np.int32)
        # clients are packed in `order` (default: index order); row_off stays per client
        order = np.arange(len(features)) if order is None else np.asarray(order, dtype=np.int64)
        self.row_off = np.zeros(len(features), dtype=np.int64)
        if len(features):
            packed_off = np.zeros(len(features), dtype=np.int64)
            packed_off[1:] = np.cumsum(n_rows[order])[:-1]
            self.row_off[order] = packed_off
        self.dim = features[0].shape[1] if features else 0
        x = (np.ascontiguousarray(np.concatenate([features[i] for i in order], axis=0), dtype=np.float64)
             if features else np.zeros((0, self.dim)))
        y = (np.ascontiguousarray(np.concatenate([np.asarray(labels[i], dtype=np.float64) for i in order]))
             if labels else np.zeros(0))
        self.x = torch.from_numpy(x.reshape(-1, self.dim) if self.dim else x)
        self.y = torch.from_numpy(y)
        self.bf16 = bf16
        if bf16:
            # the tensor-core trainer's input format, converted once like any
            # dataset preprocessing: rows zero-padded to 16 columns, features
            # rounded float64 -> float32 -> bf16 (the same two RN steps as
            # fs_prep_features_bf16), labels float32
            self.dp = (self.dim + 15) // 16 * 16
            xb = torch.zeros((self.x.shape[0], self.dp), dtype=torch.bfloat16)
            xb[:, :self.dim] = self.x.to(torch.float32).to(torch.bfloat16)
            self.x, self.y = xb, self.y.to(torch.float32)
        self.pinned = pin
        if pin:
            self.x = self.x.pin_memory()
            self.y = self.y.pin_memory()
        # upload chunks: consecutive clients of the packing order, ~chunk_bytes
        # each; chunk_of[client] tells a trainer which chunk holds its rows
        self.chunk_of = np.zeros(len(features), dtype=np.int32)
        self.chunks = [(0, int(self.x.shape[0]))]
        if chunk_bytes > 0 and len(features):
            row_bytes = self.x.element_size() * (self.x.shape[1] if self.x.dim() == 2 else 1)
            target = chunk_bytes
            bounds, start, acc = [], 0, 0
            for i in order:
                self.chunk_of[i] = len(bounds)
                acc += int(n_rows[i]) * row_bytes
                if acc >= target:
                    end = int(self.row_off[i] + n_rows[i])
                    bounds.append((start, end))
                    start, acc = end, 0
            if start < self.x.shape[0] or not bounds:
                bounds.append((start, int(self.x.shape[0])))
            self.chunks = bounds

    def to_device(self, t: torch.Tensor, rt: Runtime) -> torch.Tensor:
        if t.numel() == 0:
            return torch.empty(t.shape, dtype=t.dtype, device=rt.device)
        src = t if self.pinned else t.pin_memory()
        return src.to(rt.device, non_blocking=True)

    @property
    def nbytes(self) -> int:
        return self.x.numel() * self.x.element_size() + self.y.numel() * self.y.element_size()


class DeviceShards:
    """All client shards packed row-wise in HBM ([rows x d] float64 + labels).

    The reference keeps one numpy shard per WorldClient (server.py:89-106);
    here they are concatenated once at world build so a training launch
    addresses any client by (row offset, rows).
    """

    def __init__(self, features: list[np.ndarray], labels: list[np.ndarray], rt: Runtime | None = None,
                 packed: "HostPack | None" = None):
        self.rt = rt or Runtime.get()
        pack = packed if packed is not None else HostPack(features, labels, pin=False)
        self.n_rows, self.row_off, self.dim = pack.n_rows, pack.row_off, pack.dim
        if pack.bf16:  # bf16-only shards (tensor-core trainer input)
            self.features = self.labels = None
            self._bf16 = (pack.to_device(pack.x, self.rt), pack.to_device(pack.y, self.rt))
        else:
            self.features = pack.to_device(pack.x, self.rt)
            self.labels = pack.to_device(pack.y, self.rt)

    def __len__(self) -> int:
        return len(self.n_rows)

    def bf16(self):
        """(features bf16 [rows x round16(d)], labels fp32) for the tensor-core trainer."""
        if getattr(self, "_bf16", None) is None:
            rows = self.features.shape[0] if self.features.dim() == 2 else 0
            dp = (self.dim + 15) // 16 * 16
            xb = torch.empty((rows, dp), dtype=torch.bfloat16, device=self.rt.device)
            yf = torch.empty(rows, dtype=torch.float32, device=self.rt.device)
            self.rt.call(self.rt.lib.fs_prep_features_bf16(self.features.data_ptr(), self.labels.data_ptr(), rows,
                                                           self.dim, dp, xb.data_ptr(), yf.data_ptr(), self.rt.stream),
                         "fs_prep_features_bf16")
            self._bf16 = (xb, yf)
        return self._bf16


# --------------------------------------------------------------- training
@dataclass
class TrainRequest:
    """One local training: shard `client` from `w_start` over steps [start, end)."""

    client: int
    seed: int               # train seed (derive_seed(master, "train", cid, cycle))
    lr: np.ndarray          # [epochs] step size of each epoch
    w_start: torch.Tensor   # float64 [M] on device
    batch: int
    start_step: int = 0
    end_step: int | None = None


def steps_per_epoch(n: int, b: int) -> int:
    return -(-n // b)


def train_requests(spec_dims, shards: DeviceShards, reqs: list[TrainRequest], epochs: int,
                   dropout_rate: float, w_out: torch.Tensor | None = None,
                   rt: Runtime | None = None):
    """List-of-requests front end of :func:`train_batch` (fp64 trainer: every
    start vector must be a float64 device tensor)."""
    n = len(reqs)
    for r in reqs:
        if r.w_start.dtype != torch.float64 or not r.w_start.is_cuda:
            raise ValueError(f"w_start must be a float64 CUDA tensor, got {r.w_start.dtype} on {r.w_start.device}")
    return train_batch(
        spec_dims, shards,
        clients=np.array([r.client for r in reqs], dtype=np.int64),
        seeds=np.array([r.seed for r in reqs], dtype=np.uint64),
        lr=np.stack([np.broadcast_to(np.asarray(r.lr, dtype=np.float64), (epochs,)) for r in reqs])
        if n and epochs else np.zeros((n, max(epochs, 1))),
        w_start=np.array([r.w_start.data_ptr() for r in reqs], dtype=np.uint64),
        batch=np.array([r.batch for r in reqs], dtype=np.int64),
        epochs=epochs, dropout_rate=dropout_rate,
        start=np.array([r.start_step for r in reqs], dtype=np.int64),
        end=np.array([-1 if r.end_step is None else r.end_step for r in reqs], dtype=np.int64),
        w_out=w_out, rt=rt)


class TrainPlan:
    """The data-independent half of a training launch: per-request metadata in
    HBM plus the K2 permutations and K3 dropout keep-bits. It depends only on
    (clients, train seeds, batch sizes, epochs), never on model values, so the
    engines build the NEXT round's plan on a side stream while the current
    round's aggregation, evaluation and event bookkeeping run."""

    def __init__(self, spec_dims, shards: "DeviceShards", clients, seeds, batch, epochs: int,
                 dropout_rate: float, start=None, end=None, rt: Runtime | None = None, stream=None,
                 pool: dict | None = None, stage: "Stage | None" = None,
                 data_chunk: np.ndarray | None = None):
        rt = rt or Runtime.get()
        self.rt = rt
        self.stage = stage
        self.mask_flags = None   # per-(request, step) keep-bit flags: unused by the engines (K3 runs before the trainer)
        self._desc = None        # (precision, static TrainDesc) built by static_desc()
        self.workspace_need = 0
        self.prefilled = None    # (precision, lr, desc, w_out, status, run) prepared by prefill()
        self.opt = None          # opt-in Adam (beta1, beta2, eps); None = SGD (set before static_desc)
        self.mask_tag = 0
        lib = rt.lib
        self.dims = tuple(int(x) for x in spec_dims)
        self.shards = shards
        self.epochs = int(epochs)
        self.dropout_rate = float(dropout_rate)
        cl = np.asarray(clients, dtype=np.int64)
        n = len(cl)
        self.n = n
        self.clients = cl
        self.seeds = np.asarray(seeds, dtype=np.uint64)
        self.batch = np.asarray(batch, dtype=np.int64)
        self.ready = None
        if n == 0:
            return
        torch_stream = stream if stream is not None else torch.cuda.current_stream(rt.device)
        self.stream = torch_stream
        s_handle = torch_stream.cuda_stream
        sum_hidden = sum(self.dims[1:-1])
        n_rows = shards.n_rows[cl].astype(np.int64)
        spe = -(-n_rows // self.batch)
        total = self.epochs * spe
        start = np.zeros(n, dtype=np.int64) if start is None else np.asarray(start, dtype=np.int64)
        end = total.copy() if end is None else np.where(np.asarray(end) < 0, total, end).astype(np.int64)
        self.n_rows, self.spe, self.start, self.end = n_rows, spe, start, end
        perm_len = self.epochs * n_rows
        perm_off = np.zeros(n, dtype=np.int64)
        np.cumsum(perm_len[:-1], out=perm_off[1:])
        use_masks = self.dropout_rate > 0.0
        slot = (self.batch * sum_hidden + 31) // 32
        mask_len = total * slot if use_masks else np.zeros(n, dtype=np.int64)
        mask_off = np.zeros(n, dtype=np.int64)
        np.cumsum(mask_len[:-1], out=mask_off[1:])
        # longest client first (LPT) so the critical path starts at t=0
        order = np.argsort(-((end - start) * self.batch), kind="stable")
        def buf(name, n_elems, dtype):
            # `pool`: caller-owned buffers reused across plans (no per-round allocation)
            if pool is None:
                return torch.empty(n_elems, dtype=dtype, device=rt.device)
            t = pool.get(name)
            if t is None or t.numel() < n_elems:
                t = torch.empty(int(n_elems * 1.25) + 1, dtype=dtype, device=rt.device)
                pool[name] = t
            return t[:n_elems]

        self.pooled = pool is not None
        self._pool = pool
        with torch.cuda.stream(torch_stream):
            i64 = np.concatenate([shards.row_off[cl], perm_off, mask_off, self.seeds.view(np.int64)])
            self.has_chunks = data_chunk is not None
            parts = [n_rows, self.batch, start, end, order]
            if self.has_chunks:
                parts.append(np.asarray(data_chunk, dtype=np.int64)[cl])
            i32 = np.concatenate(parts).astype(np.int32)
            if stage is not None:
                self.d_i64 = self.d_i32 = None
                p64, p32 = stage.put(i64), stage.put(i32)
                stage.commit(torch_stream)
            else:
                self.d_i64 = buf("i64", len(i64), torch.int64)
                self.d_i32 = buf("i32", len(i32), torch.int32)
                if pool is not None:
                    # page-locked landing buffers kept in the pool: a fresh
                    # pin_memory() per plan can hit cudaHostAlloc, which waits
                    # for the whole device (a host stall in the middle of a round)
                    h64 = pool.get("h_i64")
                    if h64 is None or h64.numel() < len(i64):
                        h64 = pool["h_i64"] = torch.empty(int(len(i64) * 1.25) + 1, dtype=torch.int64).pin_memory()
                    h32 = pool.get("h_i32")
                    if h32 is None or h32.numel() < len(i32):
                        h32 = pool["h_i32"] = torch.empty(int(len(i32) * 1.25) + 1, dtype=torch.int32).pin_memory()
                    h64.numpy()[:len(i64)] = i64
                    h32.numpy()[:len(i32)] = i32
                    self.d_i64.copy_(h64[:len(i64)], non_blocking=True)
                    self.d_i32.copy_(h32[:len(i32)], non_blocking=True)
                else:
                    self.d_i64.copy_(torch.from_numpy(i64).pin_memory(), non_blocking=True)
                    self.d_i32.copy_(torch.from_numpy(i32).pin_memory(), non_blocking=True)
                p64, p32 = self.d_i64.data_ptr(), self.d_i32.data_ptr()
            self.perm = buf("perm", max(int(perm_len.sum()), 1), torch.int32)
            self.bits = (buf("bits", max(int(mask_len.sum()), 1), torch.int32)
                         if use_masks and self.epochs > 0 else None)
        self.row_off_p, self.perm_off_p, self.mask_off_p, self.seeds_p = (p64 + 8 * n * k for k in range(4))
        self.n_rows_p, self.batch_p, self.start_p, self.end_p, self.order_p = (p32 + 4 * n * k for k in range(5))
        self.chunk_p = p32 + 4 * n * 5 if self.has_chunks else None
        self.scale = 1.0
        self.max_steps = int(end.max()) if n else 0
        self.sum_hidden = sum_hidden
        keep = 1.0 - self.dropout_rate

        def launch_k2():
            if self.epochs > 0:
                rt.call(lib.fs_shuffle_perms(self.seeds_p, self.n_rows_p, self.perm_off_p, n, self.epochs,
                                             int(n_rows.max()), self.perm.data_ptr(), s_handle), "fs_shuffle_perms")

        def launch_k3():
            rt.call(lib.fs_dropout_bits(self.seeds_p, self.n_rows_p, self.batch_p, self.mask_off_p, n,
                                        self.epochs, sum_hidden, keep, self.bits.data_ptr(), s_handle),
                    "fs_dropout_bits")

        # K2 then K3 on the plan's stream (K3 first or on a second stream was
        # measured: the trainer slows by as much as the round tail gains)
        launch_k2()
        if self.bits is not None:
            launch_k3()
            self.scale = 1.0 / keep
        if stream is not None:  # consumer stream waits on this event before the trainer reads the plan
            self.ready = torch.cuda.Event()
            self.ready.record(torch_stream)

    def prefill(self, lr: float, precision: str) -> None:
        """Prepare the whole launch of a plan that one sync round will run with
        one step size: broadcast `lr` into the pooled lr buffer and zero the
        pooled status on the plan's own stream (before `ready`), and build the
        complete descriptor over pooled output rows and workspace. The round
        then launches its trainer with one fill (the start-model pointers) and
        no descriptor work. Pools alternate by round parity (engine), so a
        round's rows are dead before the same pool is prepared again."""
        if not self.pooled or self.n == 0 or self.ready is None:
            return
        lib, st = self.rt.lib, self.stream.cuda_stream
        with torch.cuda.stream(self.stream):  # allocated where written: a block the caching
            # allocator hands out on another stream may still be read by that stream's queued work
            d_lr = self.pool_buf("lr", self.n * max(self.epochs, 1), torch.float64)
            d_st = self.pool_buf("status", self.n, torch.int32)
        self.rt.call(lib.fs_fill_u64(d_lr.data_ptr(), int(np.float64(lr).view(np.uint64)), d_lr.numel(), st),
                     "fs_fill_u64")
        self.rt.call(lib.fs_fill_u64(d_st.data_ptr(), 0, (self.n + 1) // 2, st), "fs_fill_u64")
        self.ready.record(self.stream)
        # output rows and workspace: written and read by the consuming (current) stream
        bf16 = precision == "bf16"
        M = sum((a + 1) * b for a, b in zip(self.dims[:-1], self.dims[1:]))
        esz = 4 if bf16 else 8
        ld = (M * esz + 127) // 128 * 128 // esz
        w_out = self.pool_buf("w_out", self.n * ld, torch.float32 if bf16 else torch.float64).view(self.n, ld)[:, :M]
        desc = N.TrainDesc.from_buffer_copy(self.static_desc(precision))
        ws = self.pool_buf("train_ws", self.workspace_need, torch.uint8)
        d_run = self.pool_buf("run", self.n, torch.int64)
        desc.lr, desc.status = d_lr.data_ptr(), d_st.data_ptr()
        desc.w_out, desc.ldw = w_out.data_ptr(), w_out.stride(0)
        desc.workspace, desc.workspace_bytes = ws.data_ptr(), ws.numel()
        desc.w_start = d_run.data_ptr()
        if self.opt is not None:
            desc.opt_state = self.pool_buf("opt", 2 * self.n * ld, w_out.dtype).data_ptr()
        if fused_align_supported(self.dims, precision) and self.opt is None:
            # the unit-major kernel takes the one start model directly and finds
            # its work counter zeroed here: the round launches it with no fill/memset
            self.rt.call(lib.fs_fill_u64(ws.data_ptr(), 0, 1, st), "fs_fill_u64")
            self.ready.record(self.stream)
            desc.counter_zeroed = 1
        self.prefilled = (precision, float(lr), desc, w_out, d_st, d_run)

    def static_desc(self, precision: str) -> "N.TrainDesc":
        """The launch descriptor fields fixed by the plan (geometry, plan
        buffers, grid) and the trainer's workspace size, built once per plan:
        the engines call this while prefetching, off the round's critical path."""
        if self._desc is not None and self._desc[0] == precision:
            return self._desc[1]
        bf16 = precision == "bf16"
        if not bf16 and self.shards.features is None:
            raise ValueError("these shards hold bf16 features only (tensor-core trainer input)")
        desc = N.TrainDesc()
        desc.n_dims = len(self.dims)
        for i, v in enumerate(self.dims):
            desc.dims[i] = v
        desc.n_req = self.n
        desc.epochs = self.epochs
        desc.max_batch = int(self.batch.max())
        desc.max_rows = int(self.n_rows.max())
        desc.mask_mode = N.FS_MASK_BITS if self.bits is not None else N.FS_MASK_NONE
        desc.scale = self.scale
        desc.features = self.shards.features.data_ptr() if self.shards.features is not None else None
        desc.labels = self.shards.labels.data_ptr() if self.shards.labels is not None else None
        desc.row_off = self.row_off_p
        desc.n_rows = self.n_rows_p
        desc.batch = self.batch_p
        desc.perm = self.perm.data_ptr()
        desc.perm_off = self.perm_off_p
        desc.mask_bits = self.bits.data_ptr() if self.bits is not None else None
        desc.mask_off = self.mask_off_p
        desc.start_step = self.start_p
        desc.end_step = self.end_p
        desc.order = self.order_p
        desc.grid = TRAIN_GRID
        if self.opt is not None:
            desc.optimizer = N.FS_OPT_ADAM
            desc.adam_beta1, desc.adam_beta2, desc.adam_eps = (float(v) for v in self.opt)
        lib = self.rt.lib
        need = (lib.fs_train_bf16_workspace_bytes if bf16 else lib.fs_train_workspace_bytes)(ctypes.byref(desc))
        if need == 0:
            raise ValueError(f"layer dims {self.dims} are not supported by the {precision} trainer")
        self.workspace_need = need
        self._desc = (precision, desc)
        return desc

    def pool_buf(self, name: str, n_elems: int, dtype) -> torch.Tensor:
        """A pooled device buffer owned by this plan's pool (stream-ordered reuse)."""
        t = self._pool.get(name)
        if t is None or t.numel() < n_elems or t.dtype != dtype:
            t = torch.empty(int(n_elems * 1.25) + 1, dtype=dtype, device=self.rt.device)
            self._pool[name] = t
        return t[:n_elems]

    def matches(self, clients, seeds, batch, epochs) -> bool:
        return (self.epochs == epochs and np.array_equal(self.clients, clients)
                and np.array_equal(self.seeds, seeds) and np.array_equal(self.batch, batch))

    def consume(self, stream) -> None:
        """Order `stream` after the plan's producer and keep its buffers alive for it."""
        if self.ready is not None:
            stream.wait_event(self.ready)
            if not self.pooled:
                for t in (self.d_i64, self.d_i32, self.perm, self.bits):
                    if t is not None:
                        t.record_stream(stream)
            self.ready = None


def _upload_waits(plan: TrainPlan, desc, up: dict, bf16: bool, stream) -> None:
    """Order the trainer after a chunked shard upload still in flight
    (DeviceWorld.refill): per-client chunk flags for the tcgen05 trainer,
    the whole upload for the others. An upload without flags carries only
    the test set (the shards went up on the trainer's own stream)."""
    if up["flags"] is None:
        return
    if bf16 and plan.chunk_p is not None and eval_bf16_supported(plan.dims) and plan.opt is None:
        desc.data_flags = up["flags"].data_ptr()
        desc.data_chunk = plan.chunk_p
        desc.data_tag = up["tag"]
    else:
        stream.wait_event(up["done"])


def _launch_trainer(plan: TrainPlan, desc, bf16: bool, stream) -> None:
    rt, lib, dims = plan.rt, plan.rt.lib, plan.dims
    with rt.timed("train", 0.0) as tm:
        if bf16:
            xb, yf = plan.shards.bf16()
            rt.call(lib.fs_train_bf16(ctypes.byref(desc), xb.data_ptr(), yf.data_ptr(), stream.cuda_stream),
                    "fs_train_bf16")
        else:
            rt.call(lib.fs_train_f64(ctypes.byref(desc), stream.cuda_stream), "fs_train_f64")
        if tm is not None:  # algorithmic FLOPs of this launch (rows actually trained), counted after it
            s, e, spe, b, nr = plan.start, plan.end, plan.spe, plan.batch, plan.n_rows
            last = e // spe - s // spe   # epoch-final (partial) steps in [start, end)
            rows = (e - s - last) * b + last * (nr - (spe - 1) * b)
            tm.work = float(rows.sum()) * mlp_flops_per_sample(dims)


def _fused_align(plan: TrainPlan, desc, align, stream) -> None:
    """K6 fused into the unit-major trainer (fs_train_desc.align_counts):
    align = (mode, counts int64 [n] device, w_prev pointer or None)."""
    mode, counts, wprev = align
    m = N.FS_ALIGN_WEIGHT_SIGN if mode == "weight_sign" else N.FS_ALIGN_DELTA_SIGN
    desc.align_mode = m
    desc.align_counts = counts.data_ptr()
    desc.w_prev = None
    if m == N.FS_ALIGN_DELTA_SIGN:
        d_prev = plan.pool_buf("w_prev", plan.n, torch.int64) if plan.pooled else \
            torch.empty(plan.n, dtype=torch.int64, device=plan.rt.device)
        plan.rt.call(plan.rt.lib.fs_fill_u64(d_prev.data_ptr(), int(wprev), plan.n, stream.cuda_stream),
                     "fs_fill_u64")
        desc.w_prev = d_prev.data_ptr()
        plan._keep_prev = d_prev


def fused_align_supported(dims, precision: str) -> bool:
    """The trainer can count K6 itself (bf16 unit-major kernel shapes)."""
    return precision == "bf16" and eval_bf16_supported(dims)


def run_trainer(plan: TrainPlan, lr: np.ndarray, w_start: np.ndarray, precision: str = "fp64",
                w_out: torch.Tensor | None = None, status: torch.Tensor | None = None, align=None):
    """K5 over a prepared plan: lr [n x epochs], w_start [n] device pointers.
    `align` = (mode, counts [n] int64 device tensor, w_prev pointer | None):
    the trainer also writes each client's K6 count (fused_align_supported).
    Returns (w_out [n x M], status int32 [n]) on the device."""
    rt = plan.rt
    lib = rt.lib
    n = plan.n
    dims = plan.dims
    M = sum((a + 1) * b for a, b in zip(dims[:-1], dims[1:]))
    bf16 = precision == "bf16"
    pre = plan.prefilled
    up = getattr(plan.shards, "upload", None)  # a chunked upload still in flight (DeviceWorld.refill)
    if (pre is not None and pre[0] == precision and w_out is None and status is None and np.ndim(lr) == 0
            and float(lr) == pre[1] and np.ndim(w_start) == 0 and plan.mask_flags is None):
        # the launch prepared while this plan was prefetched (TrainPlan.prefill);
        # used once (its work counter is zeroed for exactly one launch)
        desc, w_out, status, d_run = pre[2], pre[3], pre[4], pre[5]
        plan.prefilled = None
        stream = torch.cuda.current_stream(rt.device)
        plan.consume(stream)
        desc.data_flags, desc.data_chunk, desc.data_tag = None, None, 0
        desc.align_counts, desc.w_prev, desc.align_mode = None, None, -1
        if up is not None and up["pending"]:
            _upload_waits(plan, desc, up, bf16, stream)
        if align is not None:
            _fused_align(plan, desc, align, stream)
        if desc.counter_zeroed:
            desc.w_start, desc.w_start_all = None, int(w_start)
        else:
            rt.call(lib.fs_fill_u64(d_run.data_ptr(), int(w_start), n, stream.cuda_stream), "fs_fill_u64")
        _launch_trainer(plan, desc, bf16, stream)
        return w_out, status
    if w_out is None:
        # rows padded to 128 bytes: 16-byte vector access to every client row
        esz = 4 if bf16 else 8
        ld = (M * esz + 127) // 128 * 128 // esz
        w_out = torch.empty((n, ld), dtype=torch.float32 if bf16 else torch.float64, device=rt.device)[:, :M]
    if bf16 and (w_out.data_ptr() % 16 or (w_out.stride(0) * 4) % 16):
        raise ValueError("bf16 trainer needs 16-byte aligned float32 rows")
    if status is None:
        status = torch.zeros(max(n, 1), dtype=torch.int32, device=rt.device)[:n]
    if n == 0:
        return w_out, status
    stream = torch.cuda.current_stream(rt.device)
    plan.consume(stream)
    if np.ndim(lr) == 0 and np.ndim(w_start) == 0 and plan.pooled:
        # one step size and one start model for the whole launch (a sync round):
        # filled on the device into the plan's pooled buffers, no host staging
        d_run = plan.pool_buf("run", n, torch.int64)
        d_lr = plan.pool_buf("lr", n * max(plan.epochs, 1), torch.float64)
        rt.call(lib.fs_fill_u64(d_run.data_ptr(), int(w_start), n, stream.cuda_stream), "fs_fill_u64")
        rt.call(lib.fs_fill_u64(d_lr.data_ptr(), int(np.float64(lr).view(np.uint64)), d_lr.numel(),
                                stream.cuda_stream), "fs_fill_u64")
        run_p, lr_p = d_run.data_ptr(), d_lr.data_ptr()
    elif plan.stage is not None:
        run_p = plan.stage.put(np.asarray(w_start, dtype=np.uint64))
        lr_p = plan.stage.put(np.ascontiguousarray(lr, dtype=np.float64).reshape(n, -1))
        plan.stage.commit(stream)
    else:
        w_arr = np.broadcast_to(np.asarray(w_start, dtype=np.uint64), (n,))
        lr_arr = np.broadcast_to(np.asarray(lr, dtype=np.float64).reshape(-1, 1) if np.ndim(lr) == 1 else
                                 np.asarray(lr, dtype=np.float64), (n, max(plan.epochs, 1)))
        d_run = rt.h2d(np.array(w_arr, dtype=np.uint64).view(np.int64))  # writable copies of the views
        d_lr = rt.h2d(np.array(lr_arr, dtype=np.float64))
        run_p, lr_p = d_run.data_ptr(), d_lr.data_ptr()
    desc = N.TrainDesc.from_buffer_copy(plan.static_desc(precision))
    desc.lr = lr_p
    desc.w_start = run_p
    desc.w_out = w_out.data_ptr()
    desc.ldw = w_out.stride(0)
    desc.status = status.data_ptr()
    if up is not None and up["pending"]:
        _upload_waits(plan, desc, up, bf16, stream)
    if align is not None:
        _fused_align(plan, desc, align, stream)
    if plan.mask_flags is not None:
        if not plan.mask_tag:
            raise ValueError("deferred keep bits need a nonzero mask_tag (the tag fs_dropout_bits_flagged publishes)")
        desc.mask_flags = plan.mask_flags.data_ptr()
        desc.mask_tag = plan.mask_tag
        desc.max_steps = plan.max_steps
    ws = rt.scratch("train", plan.workspace_need)
    desc.workspace = ws.data_ptr()
    desc.workspace_bytes = ws.numel()
    if plan.opt is not None:  # Adam moments, [n][2][ldw] of the parameter dtype, zeroed by the trainer
        desc.opt_state = rt.scratch("opt_state", 2 * n * w_out.stride(0) * w_out.element_size()).data_ptr()
    _launch_trainer(plan, desc, bf16, stream)
    return w_out, status


def train_batch(spec_dims, shards: DeviceShards, clients: np.ndarray, seeds: np.ndarray, lr: np.ndarray,
                w_start: np.ndarray, batch: np.ndarray, epochs: int, dropout_rate: float,
                start: np.ndarray | None = None, end: np.ndarray | None = None,
                w_out: torch.Tensor | None = None, rt: Runtime | None = None, precision: str = "fp64",
                opt: tuple | None = None):
    """Batched K2 -> K3 -> K5 over n requests given as arrays.

    clients [n] shard index, seeds [n] uint64 train seeds, lr [n x epochs],
    w_start [n] device pointers of the start parameters, batch [n]; optional
    start/end global step (end < 0 = all E*ceil(n_i/b_i) steps).
    precision "fp64" runs the parity trainer (float64 rows); "bf16" runs the
    tcgen05 mixed-precision trainer (float32 master rows, bf16 operands).
    Returns (w_out [n x M], status int32 [n]) on the device.
    """
    plan = TrainPlan(spec_dims, shards, clients, seeds, batch, epochs, dropout_rate, start, end, rt)
    plan.opt = opt  # opt-in Adam (beta1, beta2, eps); None = SGD
    return run_trainer(plan, lr, w_start, precision, w_out)


TRAIN_GRID = 0  # persistent trainer grid (0 = library default: one CTA per SM)


# --------------------------------------------------------------- alignment
def align_requests(wc_ptrs, wg_ptrs, wgp_ptrs, M: int, mode: str, rt: Runtime | None = None,
                   dtype: torch.dtype = torch.float64, out: torch.Tensor | None = None,
                   stage: Stage | None = None) -> torch.Tensor:
    """K6: aligned counts [n] int64 (device); dtype of the parameter vectors."""
    rt = rt or Runtime.get()
    n = len(wc_ptrs)
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.int64, device=rt.device)
    if n == 0:
        return out[:0]
    m = N.FS_ALIGN_WEIGHT_SIGN if mode == "weight_sign" else N.FS_ALIGN_DELTA_SIGN
    ptrs = [np.asarray(wc_ptrs, dtype=np.uint64).ravel(), np.asarray(wg_ptrs, dtype=np.uint64).ravel()]
    if m == N.FS_ALIGN_DELTA_SIGN:
        ptrs.append(np.asarray(wgp_ptrs, dtype=np.uint64).ravel())
    if stage is not None:
        p = stage.put(np.concatenate(ptrs))
        stage.commit()
    else:
        d = rt.h2d(np.concatenate(ptrs).view(np.int64))
        p = d.data_ptr()
    esz = 4 if dtype == torch.float32 else 8
    fn = rt.lib.fs_sign_align_f32 if esz == 4 else rt.lib.fs_sign_align_f64
    with rt.timed("align", float(esz) * M * (n + (2 if m else 1))):
        rt.call(fn(p, p + 8 * n, (p + 16 * n) if m else None, n, M, m, out.data_ptr(), rt.stream),
                "fs_sign_align")
    return out[:n]


def align_rows(w_c: torch.Tensor, wg: torch.Tensor, wgp: torch.Tensor | None, M: int, mode: str,
               rt: Runtime | None = None) -> torch.Tensor:
    """K6 for every row of a trainer output block against one (w_g, w_g_prev)."""
    rt = rt or Runtime.get()
    n = w_c.shape[0]
    out = torch.empty(max(n, 1), dtype=torch.int64, device=rt.device)
    if n == 0:
        return out[:0]
    m = N.FS_ALIGN_WEIGHT_SIGN if mode == "weight_sign" else N.FS_ALIGN_DELTA_SIGN
    esz = wg.element_size()
    stride = w_c.stride(0) * w_c.element_size()
    if (wg.data_ptr() % 16) or (m and wgp.data_ptr() % 16) or (w_c.data_ptr() % 16) or (stride % 16):
        rows = w_c.data_ptr() + np.arange(n, dtype=np.uint64) * np.uint64(stride)
        return align_shared(rows, wg, wgp, M, mode, rt)
    with rt.timed("align", float(esz) * M * (n + (2 if m else 1))):
        rt.call(rt.lib.fs_sign_align_rows(w_c.data_ptr(), stride, wg.data_ptr(), wgp.data_ptr() if m else None, n, M,
                                          m, esz, out.data_ptr(), rt.stream), "fs_sign_align_rows")
    return out[:n]


def align_shared(wc_ptrs, wg: torch.Tensor, wgp: torch.Tensor | None, M: int, mode: str,
                 rt: Runtime | None = None) -> torch.Tensor:
    """K6 for a synchronous round: all rows against the same (w_g, w_g_prev)."""
    rt = rt or Runtime.get()
    n = len(wc_ptrs)
    out = torch.empty(max(n, 1), dtype=torch.int64, device=rt.device)
    if n == 0:
        return out[:0]
    m = N.FS_ALIGN_WEIGHT_SIGN if mode == "weight_sign" else N.FS_ALIGN_DELTA_SIGN
    ptrs = np.asarray(wc_ptrs, dtype=np.uint64).ravel()
    if (wg.data_ptr() % 16) or (m and wgp.data_ptr() % 16) or np.any(ptrs % 16):
        return align_requests(ptrs, np.full(n, wg.data_ptr(), dtype=np.uint64),
                              np.full(n, wgp.data_ptr(), dtype=np.uint64) if m else None, M, mode, rt, wg.dtype)
    d = rt.h2d(ptrs.view(np.int64))
    esz = wg.element_size()
    with rt.timed("align", float(esz) * M * (n + (2 if m else 1))):
        rt.call(rt.lib.fs_sign_align_shared(d.data_ptr(), wg.data_ptr(), wgp.data_ptr() if m else None, n, M, m,
                                            esz, out.data_ptr(), rt.stream), "fs_sign_align_shared")
    return out[:n]


def cosine_shared(wc_ptrs, wg: torch.Tensor, wgp: torch.Tensor, M: int, rt: Runtime | None = None) -> torch.Tensor:
    """K6c (opt-in delta_cosine): fixed-point cosine scores [n] int64 of rows
    (device pointers) against one shared (w_g, w_g_prev)."""
    rt = rt or Runtime.get()
    n = len(wc_ptrs)
    out = torch.empty(max(n, 1), dtype=torch.int64, device=rt.device)
    if n == 0:
        return out[:0]
    d = rt.h2d(np.asarray(wc_ptrs, dtype=np.uint64).view(np.int64))
    ws = rt.scratch("cosine", rt.lib.fs_cosine_align_workspace_bytes(n))
    with rt.timed("align", float(wg.element_size()) * M * (n + 2)):
        rt.call(rt.lib.fs_cosine_align(d.data_ptr(), 0, 0, wg.data_ptr(), wgp.data_ptr(), n, M, wg.element_size(),
                                       out.data_ptr(), ws.data_ptr(), ws.numel(), rt.stream), "fs_cosine_align")
    return out[:n]


def cosine_rows(w_c: torch.Tensor, wg: torch.Tensor, wgp: torch.Tensor, M: int, rt: Runtime | None = None,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """K6c for every row of a trainer output block (base + i * stride)."""
    rt = rt or Runtime.get()
    n = w_c.shape[0]
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.int64, device=rt.device)
    if n == 0:
        return out[:0]
    ws = rt.scratch("cosine", rt.lib.fs_cosine_align_workspace_bytes(n))
    with rt.timed("align", float(wg.element_size()) * M * (n + 2)):
        rt.call(rt.lib.fs_cosine_align(None, w_c.data_ptr(), w_c.stride(0) * w_c.element_size(), wg.data_ptr(),
                                       wgp.data_ptr(), n, M, wg.element_size(), out.data_ptr(), ws.data_ptr(),
                                       ws.numel(), rt.stream), "fs_cosine_align")
    return out[:n]


# --------------------------------------------------------------- FedAvg
_N_KEYS = 4


def canonical_order_ptrs(ptrs: np.ndarray, M: int, dtype: torch.dtype, rt: Runtime, row_of=None) -> np.ndarray:
    """Order of parameter rows (device pointers) by ``values.tobytes()``
    (server.py:84). K9 gathers the leading elements as big-endian integer
    keys; rows tied on that prefix fall back to full-row byte comparison
    (``row_of(i)`` -> tensor; rare)."""
    ptrs = np.asarray(ptrs, dtype=np.uint64)
    k = len(ptrs)
    if k <= 1:
        return np.arange(k)
    nk = min(_N_KEYS, M)
    d = rt.h2d(ptrs.view(np.int64))
    keys = torch.empty(k * nk, dtype=torch.int64, device=rt.device)
    fn = rt.lib.fs_gather_sort_keys_f32 if dtype == torch.float32 else rt.lib.fs_gather_sort_keys_f64
    rt.call(fn(d.data_ptr(), k, nk, keys.data_ptr(), rt.stream), "fs_gather_sort_keys")
    kh = keys.cpu().numpy().view(np.uint64).reshape(k, nk)
    order = np.lexsort([kh[:, t] for t in range(nk - 1, -1, -1)])
    if nk == M:
        return order
    sk = kh[order]
    tie = np.all(sk[1:] == sk[:-1], axis=1)  # row i+1 ties row i on the key prefix
    if not tie.any():
        return order
    if row_of is None:
        raise ValueError("rows tie on their leading bytes: a row accessor is needed to break the tie")
    out: list[int] = []
    i = 0
    while i < k:
        j = i + 1
        while j < k and tie[j - 1]:
            j += 1
        group = [int(g) for g in order[i:j]]
        if len(group) > 1:
            full = {g: row_of(g).cpu().numpy().tobytes() for g in group}
            group = sorted(group, key=lambda g: full[g])
        out.extend(group)
        i = j
    return np.asarray(out)


def canonical_order(rows: list[torch.Tensor], M: int, rt: Runtime) -> list[int]:
    """Indices of ``rows`` (tensors) sorted by ``values.tobytes()``."""
    if len(rows) <= 1:
        return list(range(len(rows)))
    ptrs = np.array([r.data_ptr() for r in rows], dtype=np.uint64)
    return [int(i) for i in canonical_order_ptrs(ptrs, M, rows[0].dtype, rt, row_of=lambda i: rows[i])]


SORT_ON_DEVICE_MAX = 1024


def aggregate_ptrs(ptrs: np.ndarray, M: int, dtype: torch.dtype, rt: Runtime | None = None,
                   row_of=None) -> torch.Tensor:
    """K9 + K7 over raw row pointers: mean in canonical byte order. Up to 1024
    rows are ordered on the device (no host synchronisation)."""
    rt = rt or Runtime.get()
    ptrs = np.asarray(ptrs, dtype=np.uint64)
    k = len(ptrs)
    esz = 4 if dtype == torch.float32 else 8
    if 1 < k <= SORT_ON_DEVICE_MAX:
        src = rt.h2d(ptrs.view(np.int64))
        d = torch.empty(k, dtype=torch.int64, device=rt.device)
        rt.call(rt.lib.fs_canonical_order(src.data_ptr(), k, M, esz, d.data_ptr(), rt.stream), "fs_canonical_order")
    else:
        order = canonical_order_ptrs(ptrs, M, dtype, rt, row_of)
        d = rt.h2d(ptrs[order].view(np.int64))
    out = torch.empty(M, dtype=dtype, device=rt.device)
    esz = out.element_size()
    fn = rt.lib.fs_aggregate_f32 if dtype == torch.float32 else rt.lib.fs_aggregate_f64
    with rt.timed("aggregate", float(esz) * M * (k + 1)):
        rt.call(fn(d.data_ptr(), k, M, out.data_ptr(), rt.stream), "fs_aggregate")
    return out


def aggregate_jobs(jobs: list[np.ndarray], M: int, dtype: torch.dtype, rt: Runtime, stage: Stage) -> torch.Tensor:
    """K9 + K7 for many independent means in one launch pair: job j = mean of
    the rows at device pointers jobs[j] in canonical order. Returns [n_jobs x
    ld] (rows padded to 128 bytes; row j is job j's mean)."""
    n = len(jobs)
    sizes = np.array([len(j) for j in jobs], dtype=np.int64)
    esz = 4 if dtype == torch.float32 else 8
    ld = (M * esz + 127) // 128 * 128 // esz
    out = torch.empty((n, ld), dtype=dtype, device=rt.device)
    if n == 0:
        return out
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    rows = np.concatenate([np.asarray(j, dtype=np.uint64) for j in jobs])
    outp = out.data_ptr() + np.arange(n, dtype=np.uint64) * np.uint64(ld * esz)
    p_rows, p_off, p_out = stage.put(rows), stage.put(off), stage.put(outp)
    stage.commit()
    scratch = rt.scratch("agg_jobs_sorted", 8 * len(rows))
    with rt.timed("aggregate", float(esz) * M * float((sizes + 1).sum()) / n):
        rt.call(rt.lib.fs_aggregate_jobs(p_rows, p_off, n, int(sizes.max()), M, esz, scratch.data_ptr(), p_out,
                                         rt.stream), "fs_aggregate_jobs")
    return out


def aggregate_rows(rows: list[torch.Tensor], M: int, rt: Runtime | None = None) -> torch.Tensor:
    """K9 + K7: mean of k device rows in canonical byte order (server.aggregate)."""
    ptrs = np.array([r.data_ptr() for r in rows], dtype=np.uint64)
    return aggregate_ptrs(ptrs, M, rows[0].dtype, rt, row_of=lambda i: rows[i])


def aggregate_rows_weighted(rows: list[torch.Tensor], weights, M: int, rt: Runtime | None = None) -> torch.Tensor:
    """Extension: sum_i w_i x_i / sum_i w_i of k device rows in canonical byte
    order (one fs_aggregate_jobs_weighted job)."""
    rt = rt or Runtime.get()
    k = len(rows)
    dt = rows[0].dtype
    esz = rows[0].element_size()
    out = torch.empty(M, dtype=dt, device=rt.device)
    meta = np.concatenate([np.array([r.data_ptr() for r in rows], dtype=np.uint64),
                           np.array([0, k], dtype=np.uint64), np.array([out.data_ptr()], dtype=np.uint64)])
    d = rt.h2d(meta.view(np.int64))
    w = rt.h2d(np.asarray(weights, dtype=np.float64))
    scratch = rt.scratch("agg_weighted", 16 * k)
    p = d.data_ptr()
    rt.call(rt.lib.fs_aggregate_jobs_weighted(p, w.data_ptr(), p + 8 * k, 1, k, M, esz, scratch.data_ptr(),
                                              scratch.data_ptr() + 8 * k, p + 8 * (k + 2), rt.stream),
            "fs_aggregate_jobs_weighted")
    return out


# --------------------------------------------------------------- eval
def forward_probs(spec_dims, w: torch.Tensor, x: torch.Tensor, dense_masks: torch.Tensor | None = None,
                  rt: Runtime | None = None) -> torch.Tensor:
    rt = rt or Runtime.get()
    dims_c, nd = dims_array(spec_dims)
    rows = x.shape[0]
    probs = torch.empty(rows, dtype=torch.float64, device=rt.device)
    need = rt.lib.fs_forward_workspace_bytes(dims_c, nd, rows)
    ws = rt.scratch("forward", need)
    rt.call(rt.lib.fs_forward_f64(dims_c, nd, w.data_ptr(), x.data_ptr(), rows, _ptr(dense_masks),
                                  probs.data_ptr(), ws.data_ptr(), ws.numel(), rt.stream), "fs_forward_f64")
    return probs


def eval_bf16_supported(spec_dims) -> bool:
    """Layer shapes of the unit-major tensor-core kernels (fs_forward_bf16)."""
    d = list(spec_dims)
    return len(d) == 5 and d[1] in (128, 256) and d[2] == 128 and d[3] == 64 and d[0] <= 64 and d[4] == 1


def forward_probs_wide(spec_dims, w32: torch.Tensor, xb: torch.Tensor, rt: Runtime | None = None) -> torch.Tensor:
    """K8 forward, bf16 mode, layer shapes beyond the on-chip kernels (fs_forward_wide)."""
    rt = rt or Runtime.get()
    dims_c, nd = dims_array(spec_dims)
    rows = xb.shape[0]
    probs = torch.empty(rows, dtype=torch.float64, device=rt.device)
    ws = rt.scratch("forward_wide", rt.lib.fs_forward_wide_workspace_bytes(dims_c, nd, rows))
    rt.call(rt.lib.fs_forward_wide(dims_c, nd, w32.data_ptr(), xb.data_ptr(), rows, probs.data_ptr(), ws.data_ptr(),
                                   ws.numel(), rt.stream), "fs_forward_wide")
    return probs


def forward_probs_bf16(spec_dims, w32: torch.Tensor, xb: torch.Tensor, rt: Runtime | None = None) -> torch.Tensor:
    """K8 forward on the tensor cores: float64 probabilities of bf16 rows under fp32 parameters."""
    rt = rt or Runtime.get()
    dims_c, nd = dims_array(spec_dims)
    rows = xb.shape[0]
    probs = torch.empty(rows, dtype=torch.float64, device=rt.device)
    rt.call(rt.lib.fs_forward_bf16(dims_c, nd, w32.data_ptr(), xb.data_ptr(), rows, probs.data_ptr(), rt.stream),
            "fs_forward_bf16")
    return probs


def eval_counts(scores: torch.Tensor, labels_i8: torch.Tensor, threshold: float, rt: Runtime | None = None,
                f32_scores: bool = False) -> torch.Tensor:
    """K8 metrics: device int64 [3] = (#correct, 2*U_pos, n_pos). `f32_scores`:
    every score is a widened float (bf16 evaluation), ranked on float keys."""
    rt = rt or Runtime.get()
    n = scores.shape[0]
    out = torch.empty(3, dtype=torch.int64, device=rt.device)
    need = rt.lib.fs_eval_workspace_bytes(n)
    ws = rt.scratch("eval", need)
    fn = rt.lib.fs_eval_metrics_f32 if f32_scores else rt.lib.fs_eval_metrics
    rt.call(fn(scores.data_ptr(), labels_i8.data_ptr(), n, float(threshold),
               out.data_ptr(), ws.data_ptr(), ws.numel(), rt.stream), "fs_eval_metrics")
    return out


def metrics_from_counts(counts: np.ndarray, n: int) -> tuple[float, float, int, int]:
    """(accuracy, auc, n_pos, n_neg) exactly as metrics.evaluate computes them."""
    correct, twice_u, n_pos = (int(c) for c in counts[:3])
    n_neg = n - n_pos
    acc = correct / n
    if n_pos == 0 or n_neg == 0:
        raise ValueError("AUC needs at least one example of each class")
    auc = (twice_u / 2.0) / (n_pos * n_neg)
    return acc, auc, n_pos, n_neg
