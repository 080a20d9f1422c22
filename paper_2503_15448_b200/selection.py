"""Sign-alignment relevance scoring and threshold filtering of client updates.

API and semantics of pkg/src/fedsim/selection.py:1-85: relevance is the
count of positions whose 3-class signs (-, 0, +) match, ``weight_sign``
comparing sign(w_c) with sign(w_g) and ``delta_sign`` comparing
sign(w_c - w_g) with sign(w_g - w_g_prev); the ratio aligned/M is compared
with theta inclusively. Counting runs on the device (K6); the batched form
``relevance_batched`` scores every client of a round in one launch.

Opt-in extensions (off by default, never on the parity path):
``mode="delta_cosine"`` scores a client by the cosine between its update
w_c - w_g and the last global step w_g - w_g_prev (K6c, float64, carried as
the fixed-point RelevanceScore(aligned=round(cos * 2^40), total=2^40)), with
theta in [-1, 1]; ``top_k`` keeps at most k accepted clients per
synchronous round, highest score first (ties: lower client index).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .model import ParamVector

MODES = ("weight_sign", "delta_sign", "delta_cosine")
DELTA_MODES = ("delta_sign", "delta_cosine")  # need w_g_prev; unscored without it
COSINE_SCALE = 1 << 40  # fixed-point denominator of delta_cosine scores (FS_COSINE_SCALE)


def score_denominator(mode: str, M: int) -> int:
    """Denominator of the integer scores K6/K6c produce: M sign positions, or
    the cosine's fixed-point scale."""
    return COSINE_SCALE if mode == "delta_cosine" else M


@dataclass(frozen=True)
class RelevanceScore:
    aligned: int
    total: int

    @property
    def ratio(self) -> float:
        return self.aligned / self.total


@dataclass(frozen=True)
class SelectionPolicy:
    theta: float = 0.65
    mode: str = "weight_sign"
    top_k: int | None = None  # extension: at most k accepted clients per synchronous round

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        lo = -1.0 if self.mode == "delta_cosine" else 0.0
        if not lo <= self.theta <= 1.0:
            raise ValueError(f"theta must be in [{lo:g},1], got {self.theta}")
        if self.top_k is not None and (int(self.top_k) != self.top_k or self.top_k < 1):
            raise ValueError(f"top_k must be a positive integer or None, got {self.top_k!r}")


def top_k_mask(scores: np.ndarray, accept: np.ndarray, k: int | None) -> np.ndarray:
    """Of the accepted entries keep the k highest scores (ties: lower index)."""
    accept = np.asarray(accept, dtype=bool)
    if k is None or accept.sum() <= k:
        return accept
    order = np.lexsort((np.arange(len(scores)), -np.asarray(scores, dtype=np.float64)))
    rank = np.empty(len(scores), dtype=np.int64)
    rank[order] = np.arange(len(scores))
    return accept & (rank < k)


def accepts(aligned: int, total: int, theta: float) -> bool:
    """Inclusive threshold on the float64 ratio, exactly as filter_update."""
    return aligned / total >= theta


def relevance_batched(wc_rows, wg_list, wgp_list, M: int, mode: str) -> np.ndarray:
    """K6 over many clients: wc_rows / wg_list / wgp_list are device tensors
    (per request). Returns host int64 aligned counts."""
    from . import device as D

    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    rt = D.Runtime.get()
    tensors = list(wc_rows) + list(wg_list) + (list(wgp_list) if mode in DELTA_MODES else [])
    dtypes = {t.dtype for t in tensors}
    if len(dtypes) > 1 or not dtypes <= {torch.float32, torch.float64}:
        raise ValueError(f"parameter vectors must share one dtype (float32 or float64), got {sorted(map(str, dtypes))}")
    if mode == "delta_cosine":
        pairs = {(g.data_ptr(), q.data_ptr()) for g, q in zip(wg_list, wgp_list)}
        if len(pairs) != 1:
            raise ValueError("delta_cosine scores rows against one shared (w_g, w_g_prev) pair")
        out = D.cosine_shared([t.data_ptr() for t in wc_rows], wg_list[0], wgp_list[0], M, rt)
        return out.cpu().numpy()
    out = D.align_requests(
        [t.data_ptr() for t in wc_rows],
        [t.data_ptr() for t in wg_list],
        [t.data_ptr() for t in wgp_list] if mode == "delta_sign" else None,
        M, mode, rt, dtype=dtypes.pop() if dtypes else torch.float64,
    )
    return out.cpu().numpy()


def calculate_relevance(w_c: ParamVector, w_g: ParamVector, w_g_prev: ParamVector | None = None,
                        mode: str = "weight_sign") -> RelevanceScore:
    """Alignment ratio between a client vector and the global model."""
    if len(w_c) != len(w_g):
        raise ValueError(f"length mismatch: {len(w_c)} vs {len(w_g)}")
    if mode == "weight_sign":
        prev = []
    elif mode in DELTA_MODES:
        if w_g_prev is None:
            raise ValueError(f"{mode} mode requires w_g_prev")
        if len(w_g_prev) != len(w_g):
            raise ValueError("w_g_prev length mismatch")
        prev = [w_g_prev]
    else:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    # the vectors' stored dtype when they share one (bf16-mode float32 rows),
    # else float64; 3-class signs of a difference are the same either way
    vecs = [w_c, w_g] + prev
    ts = [v.device_native() for v in vecs]
    if len({t.dtype for t in ts}) > 1:
        ts = [v.device_tensor() for v in vecs]
    aligned = relevance_batched(ts[:1], ts[1:2], ts[2:], len(w_c), mode)
    return RelevanceScore(aligned=int(aligned[0]), total=score_denominator(mode, len(w_c)))


def filter_update(update, w_g: ParamVector, w_g_prev: ParamVector | None,
                  policy: SelectionPolicy) -> tuple[bool, RelevanceScore]:
    """Accept iff relevance ratio >= theta (boundary inclusive)."""
    score = calculate_relevance(update.params, w_g, w_g_prev, policy.mode)
    return score.ratio >= policy.theta, score
