"""Native event loop of the buffered asynchronous engine (C-ABI fs_async_*).

The reference runs ``FederationEngine.run_async`` (pkg/src/fedsim/server.py
:485-637) as a Python event loop that trains each client inside its
``broadcast_arrive`` handler. Here the event loop is C++ (csrc/
fs_async_engine.cpp) and knows nothing about parameters: it suspends when a
``train_done`` needs an outcome that has not been computed, listing every
deferred cycle; the caller trains and scores them in one device batch and
hands the accept flags back. Aggregations are returned as jobs (new model
version <- mean of the member cycles' updates) and window reports as
requests; the processed-event log comes back as columns and is turned into
the reference's record dicts lazily (``AsyncLogBlock``), so the replay
digest is the reference's.

``drive(world, executor, ...)`` is the generic driver: the product executor
(``server.DeviceAsyncExecutor``) runs the work on the GPU; tests plug in a
CPU checker executor to pin the event logic to the reference's golden logs.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native as N

_i32, _i64, _f64, _vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
_P32 = ctypes.POINTER(ctypes.c_int32)
_P64 = ctypes.POINTER(ctypes.c_int64)
_PF = ctypes.POINTER(ctypes.c_double)

NEED_EVAL = 1
REPORT = 2

KIND_NAMES = ("broadcast_arrive", "client_fail", "train_done", "upload_arrive", "client_recover", "checkpoint",
              "buffer_timeout", "aggregate", "run_end")
_RUN_END_REASONS = ("budget", "horizon", "cycle_cap")
_TRIGGERS = ("size", "timeout")


class AsyncWorld(ctypes.Structure):
    _fields_ = [("n_clients", _i32), ("max_cycles", _i32), ("rounds", _i32), ("k_min", _i32),
                ("budget", _i64), ("buffer_timeout_s", _f64), ("agg_cost_per_update_s", _f64),
                ("horizon_s", _f64), ("recovery_s", _f64), ("transfer_s0", _f64),
                ("cid", _vp), ("steps", _vp), ("down", _vp), ("up", _vp),
                ("plan_per_cycle", _i32), ("trains", _vp), ("failed", _vp), ("recovered", _vp),
                ("fail_off", _vp), ("span", _vp), ("n_captures", _vp), ("cap_ptr", _vp), ("cap_off", _vp),
                ("w_counts0", _i64 * 4)]


class AsyncYield(ctypes.Structure):
    _fields_ = [("n_eval", _i32), ("eval_id", _P32), ("eval_ci", _P32), ("eval_cycle", _P32),
                ("eval_version", _P32),
                ("n_jobs", _i32), ("job_version", _P32), ("job_off", _P64), ("job_member", _P32),
                ("n_reports", _i32), ("rep_i", _P64), ("rep_d", _PF), ("rep_off", _P64), ("rep_stale", _P32),
                ("now_s", _f64), ("seq", _i64), ("agg_count", _i32), ("trainings", _i64), ("stopped", _i32),
                ("transfer_s", _f64), ("w_counts", _i64 * 4),
                ("rep_w", ctypes.POINTER(ctypes.c_uint64)), ("w_g", ctypes.c_uint64), ("w_g_prev", ctypes.c_uint64),
                ("flushes", _i64), ("launches", _i64), ("diverged_client", _i32), ("diverged_cycle", _i32),
                ("host_s", _f64 * 3)]


class AsyncDevice(ctypes.Structure):
    """Mirror of fs_async_device (include/fedsim_b200.h)."""

    _fields_ = [("n_dims", _i32), ("dims", _i32 * (N.FS_MAX_LAYERS + 1)), ("epochs", _i32), ("bf16", _i32),
                ("dropout_rate", _f64), ("align_mode", _i32), ("theta", _f64), ("master_seed", ctypes.c_uint64),
                ("base_lr", _f64), ("lr_decay", _f64), ("grid", _i32), ("features", _vp), ("labels", _vp),
                ("row_off_host", _vp), ("n_rows_host", _vp), ("batch_host", _vp), ("w0", _vp), ("w0_prev", _vp),
                ("stream", _vp), ("staleness_alpha", _f64), ("rank", _i32), ("world_size", _i32),
                ("owner_host", _vp), ("exchange", _vp), ("exchange_ctx", _vp)]


# fs_async_device.exchange: sums a device float64 buffer over the ranks in place
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, _vp, _vp, _i64, _vp)


class AsyncLogView(ctypes.Structure):
    _fields_ = [("n", _i64), ("kind", ctypes.POINTER(ctypes.c_int8)), ("t", _PF), ("ci", _P32), ("cycle", _P32),
                ("a", _P64), ("b", _P64), ("x", _PF), ("l", _P64), ("n_list", _i64),
                ("list_cid", _P32), ("list_stale", _P32)]


_SIGS = {
    "fs_async_create": (_vp, [ctypes.POINTER(AsyncWorld)]),
    "fs_async_destroy": (None, [_vp]),
    "fs_async_run": (ctypes.c_int, [_vp, ctypes.POINTER(AsyncYield)]),
    "fs_async_provide": (ctypes.c_int, [_vp, _i32, _vp, _vp]),
    "fs_async_log": (ctypes.c_int, [_vp, ctypes.POINTER(AsyncLogView)]),
    "fs_async_attach_device": (ctypes.c_int, [_vp, ctypes.POINTER(AsyncDevice)]),
}


def _lib():
    lib = N.load(require_gpu=False)
    if not getattr(lib, "_fs_async_bound", False):
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        lib._fs_async_bound = True
    return lib


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def cycle_plans(world, max_cycles: int):
    """The data-independent half of every (client, cycle) of an async run,
    vectorised from server.plan_cycle (server.py:205-278 semantics): trains,
    failed, recovered, fail offset, span and the number of checkpoint
    events. Without a failure schedule the plan is per client (stride 0)."""
    cl = world.clients
    n = len(cl)
    base = np.array([wc.base_span_s for wc in cl], dtype=np.float64)
    caps = [list(wc.ckpt_capture_offsets) for wc in cl]
    cap_ptr = np.zeros(n + 1, dtype=np.int32)
    cap_ptr[1:] = np.cumsum([len(c) for c in caps])
    cap_off = np.array([o for c in caps for o in c], dtype=np.float64)
    ncap_full = np.diff(cap_ptr).astype(np.int32) if world.checkpointing else np.zeros(n, dtype=np.int32)
    if world.fail_matrix is None:
        return dict(per_cycle=0, trains=np.ones(n, np.uint8), failed=np.zeros(n, np.uint8),
                    recovered=np.zeros(n, np.uint8), fail_off=np.zeros(n), span=base.copy(),
                    n_captures=ncap_full, cap_ptr=cap_ptr, cap_off=cap_off)
    C = max_cycles
    failed = world.fail_matrix[:, :C].astype(bool)
    fail_off = np.where(failed, world.fail_offsets[:, :C].astype(np.float64) * base[:, None], 0.0)
    trains = np.ones((n, C), dtype=bool)
    recovered = np.zeros((n, C), dtype=bool)
    span = np.repeat(base[:, None], C, axis=1)
    n_captures = np.repeat(ncap_full[:, None], C, axis=1)
    if world.checkpointing:
        recovered = failed.copy()
        for ci in range(n):  # captures <= fail offset; restore + redo the lost steps
            rows = np.flatnonzero(failed[ci])
            if not len(rows):
                continue
            offs = np.asarray(caps[ci], dtype=np.float64)
            fo = fail_off[ci, rows]
            k = np.searchsorted(offs, fo, side="right") if len(offs) else np.zeros(len(rows), dtype=np.int64)
            last = np.where(k > 0, offs[np.maximum(k - 1, 0)] if len(offs) else 0.0, 0.0)
            n_captures[ci, rows] = k
            span[ci, rows] = base[ci] + world.recovery_s + (fo - last)
    else:
        trains = ~failed
        span = np.where(failed, fail_off, span)
        n_captures = np.where(failed, 0, n_captures)
    return dict(per_cycle=1, trains=trains.astype(np.uint8), failed=failed.astype(np.uint8),
                recovered=recovered.astype(np.uint8), fail_off=np.ascontiguousarray(fail_off),
                span=np.ascontiguousarray(span), n_captures=np.ascontiguousarray(n_captures, dtype=np.int32),
                cap_ptr=cap_ptr, cap_off=cap_off)


def native_supported(world) -> bool:
    """The native loop covers every world whose failure schedule spans the cycle cap."""
    C = world.rounds * world.cycle_cap
    return world.fail_matrix is None or (world.fail_matrix.shape[1] >= C and world.fail_offsets is not None
                                         and world.fail_offsets.shape[1] >= C)


class AsyncLoop:
    """One fs_async_engine (one run_async call)."""

    def __init__(self, world, horizon_s, transfer_s0: float = 0.0, window_counts=None):
        self.lib = _lib()
        cl = world.clients
        n = len(cl)
        C = world.rounds * world.cycle_cap
        plans = cycle_plans(world, C)
        self.cid = np.array([wc.profile.id for wc in cl], dtype=np.int32)
        self.steps = np.array([world.epochs * wc.steps_per_epoch for wc in cl], dtype=np.int32)
        self.down = np.array([wc.profile.down_latency_s for wc in cl], dtype=np.float64)
        self.up = np.array([wc.profile.up_latency_s for wc in cl], dtype=np.float64)
        self._keep = [self.cid, self.steps, self.down, self.up] + list(plans.values())
        w = AsyncWorld()
        w.n_clients, w.max_cycles, w.rounds, w.k_min = n, C, world.rounds, int(world.k_min)
        w.budget = world.update_budget
        w.buffer_timeout_s = float(world.buffer_timeout_s)
        w.agg_cost_per_update_s = float(world.agg_cost_per_update_s)
        w.horizon_s = -1.0 if horizon_s is None else float(horizon_s)
        w.recovery_s = float(world.recovery_s)
        w.transfer_s0 = float(transfer_s0)
        w.cid, w.steps = self.cid.ctypes.data, self.steps.ctypes.data
        w.down, w.up = self.down.ctypes.data, self.up.ctypes.data
        w.plan_per_cycle = plans["per_cycle"]
        for name in ("trains", "failed", "recovered", "fail_off", "span", "n_captures", "cap_ptr", "cap_off"):
            setattr(w, name, plans[name].ctypes.data if plans[name].size else None)
        wc0 = window_counts or {}
        for i, key in enumerate(("accepted", "rejected", "failures", "steps")):
            w.w_counts0[i] = int(wc0.get(key, 0))
        self._world_struct = w
        self.handle = self.lib.fs_async_create(ctypes.byref(w))
        if not self.handle:
            raise ValueError("fs_async_create: invalid async world")
        self.y = AsyncYield()

    def attach_device(self, dev: AsyncDevice, keep=()) -> None:
        """Device mode: the engine trains, scores and aggregates on the GPU itself."""
        self._dev_struct, self._dev_keep = dev, list(keep)
        N.check(self.lib.fs_async_attach_device(self.handle, ctypes.byref(dev)), "fs_async_attach_device")

    def run(self) -> int:
        rc = self.lib.fs_async_run(self.handle, ctypes.byref(self.y))
        if rc == N.FS_EDIVERGED:
            from .model import TrainingDivergedError

            raise TrainingDivergedError(self.lib.fs_last_error().decode(errors="replace"))
        if rc < 0:
            N.check(rc, "fs_async_run")
        return rc

    def report_versions(self) -> list[int]:
        y = self.y
        return [int(y.rep_w[i]) for i in range(y.n_reports)]

    def pending(self):
        y = self.y
        n = y.n_eval
        return (_arr(y.eval_id, n, np.int64), _arr(y.eval_ci, n, np.int64), _arr(y.eval_cycle, n, np.int64),
                _arr(y.eval_version, n, np.int64))

    def jobs(self):
        """[(version, member deferred ids)] queued since the last run() call, in order."""
        y = self.y
        if y.n_jobs == 0:
            return []
        off = _arr(y.job_off, y.n_jobs + 1, np.int64)
        mem = _arr(y.job_member, int(off[-1]), np.int64)
        ver = _arr(y.job_version, y.n_jobs, np.int64)
        return [(int(ver[j]), mem[off[j]:off[j + 1]]) for j in range(y.n_jobs)]

    def reports(self):
        y = self.y
        out = []
        if y.n_reports == 0:
            return out
        ri = _arr(y.rep_i, 9 * y.n_reports, np.int64).reshape(-1, 9)
        rd = _arr(y.rep_d, 2 * y.n_reports, np.float64).reshape(-1, 2)
        off = _arr(y.rep_off, y.n_reports + 1, np.int64)
        st = _arr(y.rep_stale, int(off[-1]), np.int64)
        for r in range(y.n_reports):
            out.append(dict(window=int(ri[r, 0]), version=int(ri[r, 1]), updates=int(ri[r, 2]),
                            aggregations=int(ri[r, 3]), accepted=int(ri[r, 4]), rejected=int(ri[r, 5]),
                            failures=int(ri[r, 6]), steps=int(ri[r, 7]), t_s=float(rd[r, 0]),
                            transfer_s=float(rd[r, 1]), staleness=st[off[r]:off[r + 1]].tolist()))
        return out

    def provide(self, accepted: np.ndarray, relevance: np.ndarray) -> None:
        acc = np.ascontiguousarray(accepted, dtype=np.uint8)
        rel = np.ascontiguousarray(relevance, dtype=np.float64)
        rc = self.lib.fs_async_provide(self.handle, len(acc), acc.ctypes.data, rel.ctypes.data)
        if rc != 0:
            raise ValueError("fs_async_provide: outcome count does not match the pending batch")

    def log_block(self) -> "AsyncLogBlock":
        v = AsyncLogView()
        self.lib.fs_async_log(self.handle, ctypes.byref(v))
        n = v.n
        cols = dict(kind=_arr(v.kind, n, np.int8), t=_arr(v.t, n, np.float64), ci=_arr(v.ci, n, np.int32),
                    cycle=_arr(v.cycle, n, np.int32), a=_arr(v.a, n, np.int64), b=_arr(v.b, n, np.int64),
                    x=_arr(v.x, n, np.float64), l=_arr(v.l, n, np.int64),
                    list_cid=_arr(v.list_cid, v.n_list, np.int64), list_stale=_arr(v.list_stale, v.n_list, np.int64))
        return AsyncLogBlock(cols, self.cid.tolist(), self.down.tolist(), self.up.tolist(), self.steps.tolist())

    def close(self) -> None:
        if self.handle:
            self.lib.fs_async_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class AsyncLogBlock:
    """The native loop's processed events, columnar; ``records()`` yields the
    reference's record dicts (server.py:530-624 payloads) in log order."""

    __slots__ = ("c", "cid", "down", "up", "steps")

    def __init__(self, cols, cid, down, up, steps):
        self.c, self.cid, self.down, self.up, self.steps = cols, cid, down, up, steps

    def __len__(self) -> int:
        return len(self.c["kind"])

    def aggregates(self):
        """(round, accepted ids, t_s) of every aggregate record, in order."""
        c = self.c
        out = []
        lc = c["list_cid"].tolist()
        for i in np.flatnonzero(c["kind"] == 7).tolist():
            l0, cnt = int(c["l"][i]), int(c["cycle"][i])
            out.append((int(c["a"][i]), lc[l0:l0 + cnt], float(c["t"][i])))
        return out

    def records(self) -> list[dict]:
        c = self.c
        cid, down, up, steps = self.cid, self.down, self.up, self.steps
        lc, ls = c["list_cid"].tolist(), c["list_stale"].tolist()
        out = []
        for k, t, ci, cy, a, b, x, l in zip(c["kind"].tolist(), c["t"].tolist(), c["ci"].tolist(),
                                            c["cycle"].tolist(), c["a"].tolist(), c["b"].tolist(),
                                            c["x"].tolist(), c["l"].tolist()):
            if k == 0:
                out.append({"t_s": t, "kind": "broadcast_arrive", "client_id": cid[ci], "round": cy,
                            "latency_s": down[ci]})
            elif k == 2:
                out.append({"t_s": t, "kind": "train_done", "client_id": cid[ci], "round": cy, "accepted": bool(a),
                            "relevance": None if math.isnan(x) else x, "steps": steps[ci]})
            elif k == 3:
                out.append({"t_s": t, "kind": "upload_arrive", "client_id": cid[ci], "round": cy,
                            "latency_s": up[ci], "staleness": a})
            elif k == 7:
                out.append({"t_s": t, "kind": "aggregate", "round": a, "window": b, "accepted_ids": lc[l:l + cy],
                            "count": cy, "cost_s": x, "trigger": _TRIGGERS[ci], "staleness": ls[l:l + cy]})
            elif k == 6:
                out.append({"t_s": t, "kind": "buffer_timeout", "epoch": a, "pending": b})
            elif k == 1:
                out.append({"t_s": t, "kind": "client_fail", "client_id": cid[ci], "round": cy, "recovered": bool(a)})
            elif k == 4:
                out.append({"t_s": t, "kind": "client_recover", "client_id": cid[ci], "round": cy})
            elif k == 5:
                out.append({"t_s": t, "kind": "checkpoint", "client_id": cid[ci], "round": cy,
                            "scope": f"client-{cid[ci]}"})
            else:
                out.append({"t_s": t, "kind": "run_end", "reason": _RUN_END_REASONS[a]})
        return out


def drive(world, executor, horizon_s=None, transfer_s0: float = 0.0, window_counts=None):
    """Run the native async loop to completion with `executor` doing the
    parameter work. The executor implements:

    * ``aggregate(version, member_ids)`` -- new model version = mean of the
      members' updates (canonical order), launched in job order;
    * ``report(info)`` -- evaluate the given version for a window report;
    * ``train(ids, ci, cycle, version) -> (accepted bool[n], relevance f64[n])``
      -- train + score a deferred batch (relevance NaN when not scored).

    Returns (loop, final yield)."""
    loop = AsyncLoop(world, horizon_s, transfer_s0, window_counts)
    while True:
        rc = loop.run()
        jobs = loop.jobs()
        if jobs and hasattr(executor, "aggregate_jobs"):
            executor.aggregate_jobs(jobs)
        else:
            for version, members in jobs:
                executor.aggregate(version, members)
        for info in loop.reports():
            executor.report(info)
        if rc != NEED_EVAL:
            break
        ids, ci, cyc, ver = loop.pending()
        accepted, relevance = executor.train(ids, ci, cyc, ver)
        loop.provide(accepted, relevance)
    return loop, loop.y
