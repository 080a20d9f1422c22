"""numpy restatement of the reference round loop (TEST INFRASTRUCTURE ONLY).

See oracle/__init__.py for the rules. Each function cites the reference
code it restates. Inputs are a ``World``-shaped object (clients with
features/labels/batch_size/profile/geometry, policy, hyper-parameters) —
built by the package's host-side world builder, whose output is itself
pinned against the reference by digest (tests/golden/worlds.json).
"""

from __future__ import annotations

import hashlib
import heapq
import json
import math

import numpy as np

# ------------------------------------------------------------------ streams
# rng.py:18-44 — a stream is SeedSequence(master, spawn_key=label words)


def stream_word(label) -> int:
    if isinstance(label, str):
        return int.from_bytes(hashlib.blake2b(label.encode(), digest_size=4).digest(), "little")
    return int(label) & 0xFFFFFFFF


def sub_seed(master: int, *path) -> int:
    ss = np.random.SeedSequence(int(master), spawn_key=tuple(stream_word(p) for p in path))
    return int(ss.generate_state(1, np.uint64)[0])


def sub_rng(master: int, *path) -> np.random.Generator:
    return np.random.default_rng(
        np.random.SeedSequence(int(master), spawn_key=tuple(stream_word(p) for p in path)))


# ------------------------------------------------------------------ MLP kernels
# numpy_backend.py:23-109 (flat float64 layout, relu, inverted dropout,
# single sigmoid unit, mean BCE from logits)


def layer_views(theta: np.ndarray, dims) -> list:
    out, at = [], 0
    for a, b in zip(dims[:-1], dims[1:]):
        W = theta[at:at + a * b].reshape(a, b)
        at += a * b
        out.append((W, theta[at:at + b]))
        at += b
    if at != theta.shape[0]:
        raise ValueError("parameter length does not match the layer dims")
    return out


def stable_sigmoid(z: np.ndarray) -> np.ndarray:  # numpy_backend.py:38-44
    out = np.empty_like(z)
    nonneg = z >= 0
    out[nonneg] = 1.0 / (1.0 + np.exp(-z[nonneg]))
    e = np.exp(z[~nonneg])
    out[~nonneg] = e / (1.0 + e)
    return out


def probs(theta, dims, x, masks=None) -> np.ndarray:  # numpy_backend.py:47-57
    layers = layer_views(theta, dims)
    h = x
    for i, (W, b) in enumerate(layers[:-1]):
        h = np.maximum(h @ W + b, 0.0)
        if masks is not None:
            h = h * masks[i]
    W, b = layers[-1]
    return stable_sigmoid((h @ W + b)[:, 0])


def bce_grad(theta, dims, x, y, masks=None):  # numpy_backend.py:60-104
    layers = layer_views(theta, dims)
    rows = x.shape[0]
    acts, pres = [x], []
    h = x
    for i, (W, b) in enumerate(layers[:-1]):
        z = h @ W + b
        pres.append(z)
        h = np.maximum(z, 0.0)
        if masks is not None:
            h = h * masks[i]
        acts.append(h)
    W_out, b_out = layers[-1]
    logit = (h @ W_out + b_out)[:, 0]
    loss = float(np.mean(np.maximum(logit, 0.0) - logit * y + np.log1p(np.exp(-np.abs(logit)))))
    grad = np.zeros_like(theta)
    g_layers = layer_views(grad, dims)
    dz = (stable_sigmoid(logit) - y) / rows
    g_layers[-1][0][:, 0] = acts[-1].T @ dz
    g_layers[-1][1][0] = dz.sum()
    delta = np.outer(dz, W_out[:, 0])
    for i in range(len(layers) - 2, -1, -1):
        d = delta if masks is None else delta * masks[i]
        d = d * (pres[i] > 0.0)
        g_layers[i][0][...] = acts[i].T @ d
        g_layers[i][1][...] = d.sum(axis=0)
        if i > 0:
            delta = d @ layers[i][0].T
    return loss, grad


def sign_matches(a, b) -> int:  # numpy_backend.py:107-109, _core.pyx:222-236
    return int(np.count_nonzero(np.sign(a) == np.sign(b)))


def keep_masks(hidden, rate, rows, seed):  # model.py:153-166
    if rate == 0.0:
        return None
    g = np.random.default_rng(np.random.SeedSequence(int(seed)))
    keep = 1.0 - rate
    return [(g.random((rows, h)) < keep).astype(np.float64) * (1.0 / keep) for h in hidden]


# ------------------------------------------------------------------ local SGD
# client.py:98-172 (+ model.loss_and_grad / sgd_step, model.py:189-221)


def local_sgd(dims, rate, w0, X, Y, epochs, bsz, lr_of_epoch, seed, stop=None, resume=None, adam=None):
    """Returns dict(params, steps, epoch, batch, samples, stopped).

    adam = (beta1, beta2, eps) selects the framework's opt-in Adam (not in
    the reference): moments from zero, t = step + 1,
    p -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)."""
    n = X.shape[0]
    hidden = dims[1:-1]
    theta = w0 if resume is None else resume["params"]
    steps = 0 if resume is None else resume["steps"]
    samples = 0 if resume is None else resume["samples"]
    e0 = 0 if resume is None else resume["epoch"]
    b0 = 0 if resume is None else resume["batch"]
    per_epoch = math.ceil(n / bsz)
    if adam is not None:
        b1, b2, eps = adam
        m1, m2 = np.zeros_like(theta), np.zeros_like(theta)
    for e in range(e0, epochs):
        order = sub_rng(seed, "shuffle", e).permutation(n)
        lr = lr_of_epoch(e)
        for s in range(b0 if e == e0 else 0, per_epoch):
            if stop is not None and steps >= stop:
                return dict(params=theta, steps=steps, epoch=e, batch=s, samples=samples, stopped=True)
            pick = order[s * bsz:(s + 1) * bsz]
            xb = np.ascontiguousarray(X[pick], dtype=np.float64)
            yb = Y[pick].astype(np.float64)
            masks = keep_masks(hidden, rate, len(pick), sub_seed(seed, "mask", e, s)) if rate > 0.0 else None
            loss, g = bce_grad(theta, dims, xb, yb, masks)
            if not np.isfinite(loss):
                raise FloatingPointError("loss became non-finite")
            if adam is None:
                theta = theta - lr * g
            else:
                t = e * per_epoch + s + 1
                m1 = b1 * m1 + (1.0 - b1) * g
                m2 = b2 * m2 + (1.0 - b2) * g * g
                theta = theta - lr * (m1 * (1.0 / (1.0 - b1 ** t))) / (np.sqrt(m2 * (1.0 / (1.0 - b2 ** t))) + eps)
            steps += 1
            samples += len(pick)
    if stop is not None and steps >= stop:
        return dict(params=theta, steps=steps, epoch=epochs, batch=0, samples=samples, stopped=True)
    return dict(params=theta, steps=steps, epoch=epochs, batch=0, samples=samples, stopped=False)


# ------------------------------------------------------------------ selection / FedAvg


COSINE_SCALE = 1 << 40  # fixed point of the opt-in delta_cosine score (framework extension)


def alignment(wc, wg, wgp, mode) -> int:  # selection.py:53-74
    if mode == "weight_sign":
        return sign_matches(wc, wg)
    if mode == "delta_cosine":  # extension (not in the reference): cos(wc - wg, wg - wgp) as llrint(cos * 2^40)
        a, b = wc - wg, wg - wgp
        na, nb = float(a @ a), float(b @ b)
        cs = min(1.0, max(-1.0, float(a @ b) / np.sqrt(na * nb))) if na > 0 and nb > 0 else 0.0
        return int(np.rint(cs * COSINE_SCALE))
    return sign_matches(wc - wg, wg - wgp)


def score_den(mode, M) -> int:
    return COSINE_SCALE if mode == "delta_cosine" else M


def top_k_keep(outs, k):
    """Extension: of the accepted scored cycles keep the k highest relevances
    (ties: lower client index); the others become rejected."""
    cand = [i for i, o in enumerate(outs) if o["res"] is not None and o["rel"] is not None and o["accepted"]]
    cand.sort(key=lambda i: (-outs[i]["rel"], i))
    for i in cand[k:]:
        outs[i]["accepted"] = False


def fedavg(vectors, weights=None):  # server.py:72-86
    if not vectors:
        return None
    ranked = sorted(range(len(vectors)), key=lambda i: vectors[i].tobytes())
    if weights is None:
        return np.stack([vectors[i] for i in ranked]).mean(axis=0)
    # extension (not in the reference): weighted mean in the same canonical
    # order, sum_i w_i x_i / sum_i w_i, sequential float64, product and sum
    # rounded separately (the kernel's __dmul_rn / __dadd_rn chain)
    acc = np.full(len(vectors[0]), -0.0)
    den = -0.0
    for i in ranked:
        acc = acc + weights[i] * vectors[i]
        den += weights[i]
    return acc / den


# ------------------------------------------------------------------ metrics
# metrics.py:118-165


def acc_auc(scores, labels, thr=0.5):
    scores = np.asarray(scores, dtype=np.float64)
    pos = np.asarray(labels) == 1
    acc = float(np.mean((scores >= thr) == pos))
    order = np.argsort(scores, kind="stable")
    ranks = np.empty(len(scores))
    srt = scores[order]
    i = 0
    while i < len(srt):
        j = i
        while j + 1 < len(srt) and srt[j + 1] == srt[i]:
            j += 1
        ranks[order[i:j + 1]] = 0.5 * (i + j) + 1.0
        i = j + 1
    n_pos = int(pos.sum())
    n_neg = len(scores) - n_pos
    u = float(np.sum(ranks[pos])) - n_pos * (n_pos + 1) / 2.0
    return acc, u / (n_pos * n_neg)


# ------------------------------------------------------------------ engines
# server.py:196-645: the client cycle, sync barrier rounds and the buffered
# async engine, on a (t, seq) event heap (simnet.py:40-97).


class _Clock:
    def __init__(self):
        self.now = 0.0
        self.q = []
        self.n = 0
        self.log = []
        self.halted = False

    def at(self, t, kind, **payload):
        if t < self.now:
            raise ValueError("event scheduled in the past")
        heapq.heappush(self.q, (float(t), self.n, kind, payload))
        self.n += 1

    def drain(self, on_event, horizon=None):
        while self.q and not self.halted:
            if horizon is not None and self.q[0][0] > horizon:
                break
            t, _, kind, payload = heapq.heappop(self.q)
            self.now = t
            rec = on_event(t, kind, payload)
            if rec is not None:
                self.log.append(rec)
        if horizon is not None and not self.halted:
            self.now = max(self.now, horizon)

    def digest(self):
        h = hashlib.blake2b(digest_size=8)
        for rec in self.log:
            h.update(json.dumps(rec, sort_keys=True).encode("utf-8"))
            h.update(b"\n")
        return h.hexdigest()


def _entry(t, kind, payload):
    rec = {"t_s": t, "kind": kind}
    rec.update(payload)
    return rec


class OracleFederation:
    """Reference semantics of FederationEngine on a world (CPU, serial)."""

    def __init__(self, world):
        self.w = world
        self.clock = _Clock()
        self.transfer = 0.0
        self.reports = []
        self.counts = dict(accepted=0, rejected=0, failures=0, steps=0)
        self.aligned_log = []   # (cycle, client, aligned) per scored training
        self.trainings = 0

    # server.py:196-301
    def cycle(self, ci, cyc, lr_round, wg, wgp):
        w = self.w
        wc = w.clients[ci]
        cid = wc.profile.id
        seed = sub_seed(w.master_seed, "train", cid, cyc)
        lr = w.base_lr * w.lr_decay ** lr_round
        span0 = wc.base_span_s
        failed = bool(w.fail_matrix[ci, cyc]) if w.fail_matrix is not None else False
        f_off = float(w.fail_offsets[ci, cyc]) * span0 if failed else None
        dims = w.spec.dims
        rate = w.spec.dropout_rate

        def train(**kw):
            return local_sgd(dims, rate, wg, wc.features, wc.labels, w.epochs, wc.batch_size,
                             lambda e: lr, seed, adam=(tuple(w.adam) if getattr(w, "optimizer", "sgd") == "adam"
                                                       else None), **kw)

        captures, redo, recovered = [], 0.0, False
        if not failed:
            captures = list(wc.ckpt_capture_offsets) if w.checkpointing else []
            res, span = train(), span0
        elif w.checkpointing:
            last_step, last_off = 0, 0.0
            for st, off in zip(wc.ckpt_capture_steps, wc.ckpt_capture_offsets):
                if off > f_off:
                    break
                last_step, last_off = st, off
            captures = [o for o in wc.ckpt_capture_offsets if o <= f_off]
            part = train(stop=last_step)
            res = train(resume=part)
            redo = f_off - last_off
            span = span0 + w.recovery_s + redo
            recovered = True
        else:
            res, span = None, f_off
        accepted, rel = False, None
        if res is not None:
            if w.policy.mode in ("delta_sign", "delta_cosine") and wgp is None:
                accepted = True
            else:
                a = alignment(res["params"], wg, wgp, w.policy.mode)
                self.aligned_log.append((cyc, cid, a))
                rel = a / score_den(w.policy.mode, len(wg))
                accepted = rel >= w.policy.theta
        return dict(cid=cid, cyc=cyc, failed=failed, recovered=recovered, f_off=f_off, span=span,
                    res=res, accepted=accepted, rel=rel, captures=captures)

    def _post_cycle(self, t0, o, label):  # server.py:366-386
        c = self.clock
        for off in o["captures"]:
            c.at(t0 + off, "checkpoint", client_id=o["cid"], round=label, scope=f"client-{o['cid']}")
        if o["failed"]:
            c.at(t0 + o["f_off"], "client_fail", client_id=o["cid"], round=label, recovered=o["recovered"])
            if o["recovered"]:
                c.at(t0 + o["f_off"] + self.w.recovery_s, "client_recover", client_id=o["cid"], round=label)
        if o["res"] is not None:
            c.at(t0 + o["span"], "train_done", client_id=o["cid"], round=label, accepted=o["accepted"],
                 relevance=o["rel"], steps=o["res"]["steps"])

    def _report(self, wg, window, t, updates, aggs, stale):  # server.py:321-353
        w = self.w
        p = probs(wg, w.spec.dims, np.ascontiguousarray(w.test_features, dtype=np.float64))
        acc, auc = acc_auc(p, w.test_labels, w.eval_threshold)
        k = self.counts
        dec = k["accepted"] + k["rejected"]
        self.reports.append(dict(round=window, t_s=t, accuracy=acc, auc=auc, updates=updates,
                                 aggregations=aggs, accepted=k["accepted"], rejected=k["rejected"],
                                 failures=k["failures"], accepted_frac=k["accepted"] / dec if dec else 0.0,
                                 staleness_mean=float(np.mean(stale)) if stale else 0.0,
                                 staleness_max=int(max(stale)) if stale else 0, sgd_steps=k["steps"]))
        self.counts = dict(accepted=0, rejected=0, failures=0, steps=0)

    # server.py:396-481
    def sync_round(self, r, wg, wgp):
        w, c = self.w, self.clock
        t0 = c.now
        arr = []
        for wc in w.clients:
            t = t0 + wc.profile.down_latency_s
            arr.append(t)
            c.at(t, "broadcast_arrive", client_id=wc.profile.id, round=r, latency_s=wc.profile.down_latency_s)
            self.transfer += wc.profile.down_latency_s
        outs = [self.cycle(ci, r, r, wg, wgp) for ci in range(len(w.clients))]
        if getattr(w.policy, "top_k", None) is not None:
            top_k_keep(outs, w.policy.top_k)
        kept, ends = [], []
        for t, o in zip(arr, outs):
            self._post_cycle(t, o, r)
            if o["res"] is None:
                self.counts["failures"] += 1
                continue
            self.trainings += 1
            if o["failed"]:
                self.counts["failures"] += 1
            done = t + o["span"]
            self.counts["steps"] += o["res"]["steps"]
            if o["accepted"]:
                up = w.clients[o["cid"]].profile.up_latency_s
                c.at(done + up, "upload_arrive", client_id=o["cid"], round=r, latency_s=up, staleness=0)
                self.transfer += up
                kept.append(o)
                ends.append(done + up)
                self.counts["accepted"] += 1
            else:
                ends.append(done)
                self.counts["rejected"] += 1
        if not ends:
            barrier = max((t + o["f_off"] for t, o in zip(arr, outs) if o["failed"]), default=t0)
            c.drain(_entry)
            c.at(barrier, "round_stalled", round=r)
            c.drain(_entry)
            self._report(wg, r, barrier, 0, 0, [])
            return wg, wgp  # stalled round: global state untouched (server.py:442-453)
        barrier = max(ends)
        cost = w.agg_cost_per_update_s * len(kept)
        c.drain(_entry)
        c.at(barrier + cost, "aggregate", round=r, window=r, accepted_ids=[o["cid"] for o in kept],
             count=len(kept), cost_s=cost, barrier_t_s=barrier)
        c.drain(_entry)
        mean = fedavg([o["res"]["params"] for o in kept])
        new = mean if mean is not None else wg
        self._report(new, r, barrier + cost, len(kept), 1, [0] * len(kept))
        return new, wg

    def run_sync(self, w0):
        wg, wgp = w0, None
        for r in range(self.w.rounds):
            wg, wgp = self.sync_round(r, wg, wgp)
        self.clock.at(self.clock.now, "run_end", reason="rounds_done")
        self.clock.drain(_entry)
        return wg

    # server.py:485-637
    def run_async(self, w0, horizon=None):
        w, c = self.w, self.clock
        n = len(w.clients)
        g = dict(wg=w0, wgp=None, aggs=0, applied=0, free=0.0, reported=0)
        cycles = [0] * n
        stale_win = []
        pending, inflight = [], {}
        buf_epoch = [0]
        cap = w.rounds * w.cycle_cap
        idx = {wc.profile.id: ci for ci, wc in enumerate(w.clients)}

        def begin(cid, t_req):
            ci = idx[cid]
            if cycles[ci] >= cap:
                return
            k = cycles[ci]
            cycles[ci] += 1
            down = w.clients[ci].profile.down_latency_s
            c.at(max(t_req, g["free"]) + down, "broadcast_arrive", client_id=cid, round=k, latency_s=down)
            self.transfer += down

        def flush(t, why):
            batch = list(pending)
            pending.clear()
            buf_epoch[0] += 1
            cost = w.agg_cost_per_update_s * len(batch)
            done = max(t, g["free"]) + cost
            g["free"] = done
            c.at(done, "aggregate", round=g["aggs"], window=g["applied"] // n,
                 accepted_ids=[u["cid"] for u, _ in batch], count=len(batch), cost_s=cost, trigger=why,
                 batch=batch)

        def on_event(t, kind, p):
            if kind == "broadcast_arrive":
                cid, k = p["client_id"], p["round"]
                o = self.cycle(idx[cid], k, min(k, w.rounds - 1), g["wg"], g["wgp"])
                self._post_cycle(t, o, k)
                if o["res"] is None:
                    self.counts["failures"] += 1
                    begin(cid, t + o["span"])
                else:
                    if o["failed"]:
                        self.counts["failures"] += 1
                    inflight[(cid, k)] = (o, g["aggs"])
                return _entry(t, kind, p)
            if kind == "train_done":
                o, fetched = inflight.pop((p["client_id"], p["round"]))
                self.trainings += 1
                self.counts["steps"] += o["res"]["steps"]
                if o["accepted"]:
                    self.counts["accepted"] += 1
                    up = w.clients[idx[o["cid"]]].profile.up_latency_s
                    c.at(t + up, "upload_arrive", client_id=o["cid"], round=p["round"], latency_s=up,
                         staleness=None, update=o, fetched=fetched)
                    self.transfer += up
                else:
                    self.counts["rejected"] += 1
                    begin(o["cid"], t)
                return _entry(t, kind, p)
            if kind == "upload_arrive":
                o, fetched = p.pop("update"), p.pop("fetched")
                pending.append((o, fetched))
                if len(pending) == 1:
                    c.at(t + w.buffer_timeout_s, "buffer_timeout", epoch=buf_epoch[0], pending=1)
                if len(pending) >= w.k_min:
                    flush(t, "size")
                begin(p["client_id"], t)
                rec = _entry(t, kind, p)
                rec["staleness"] = g["aggs"] - fetched
                return rec
            if kind == "buffer_timeout":
                if p["epoch"] != buf_epoch[0]:
                    return None
                if pending:
                    flush(t, "timeout")
                return _entry(t, kind, p)
            if kind == "aggregate":
                batch = p.pop("batch")
                stale = [g["aggs"] - f for _, f in batch]
                alpha = getattr(w, "staleness_alpha", None)
                wts = None if alpha is None else [(1.0 + s) ** -alpha for s in stale]
                mean = fedavg([u["res"]["params"] for u, _ in batch], wts)
                g["wgp"] = g["wg"]
                if mean is not None:
                    g["wg"] = mean
                g["aggs"] += 1
                before = g["applied"]
                g["applied"] += len(batch)
                stale_win.extend(stale)
                rec = _entry(t, kind, p)
                rec["staleness"] = stale
                for win in range(before // n, min(g["applied"] // n, w.rounds)):
                    self._report(g["wg"], win, t, n, g["aggs"] - g["reported"], list(stale_win))
                    g["reported"] = g["aggs"]
                    stale_win.clear()
                if g["applied"] >= w.rounds * n:
                    c.at(t, "run_end", reason="budget")
                return rec
            if kind == "run_end":
                c.halted = True
                return _entry(t, kind, p)
            return _entry(t, kind, p)

        for wc in w.clients:
            begin(wc.profile.id, 0.0)
        horizon = horizon if horizon is not None else w.horizon_s
        c.drain(on_event, horizon)
        if not c.halted:
            why = "horizon" if horizon is not None and c.now >= horizon else "cycle_cap"
            c.at(c.now, "run_end", reason=why)
            c.drain(on_event)
        return g["wg"]

    def run(self, w0):
        if self.w.mode in ("sync_baseline", "sync_filtered"):
            return self.run_sync(w0)
        return self.run_async(w0)

    def digest(self):
        return self.clock.digest()
