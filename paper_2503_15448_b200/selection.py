"""Sign-alignment relevance scoring and threshold filtering of client updates.

API and semantics of pkg/src/fedsim/selection.py:1-85: relevance is the
count of positions whose 3-class signs (-, 0, +) match, ``weight_sign``
comparing sign(w_c) with sign(w_g) and ``delta_sign`` comparing
sign(w_c - w_g) with sign(w_g - w_g_prev); the ratio aligned/M is compared
with theta inclusively. Counting runs on the device (K6); the batched form
``relevance_batched`` scores every client of a round in one launch.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .model import ParamVector

MODES = ("weight_sign", "delta_sign")


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

    def __post_init__(self):
        if not 0.0 <= self.theta <= 1.0:
            raise ValueError(f"theta must be in [0,1], got {self.theta}")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")


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
    tensors = list(wc_rows) + list(wg_list) + (list(wgp_list) if mode == "delta_sign" else [])
    dtypes = {t.dtype for t in tensors}
    if len(dtypes) > 1 or not dtypes <= {torch.float32, torch.float64}:
        raise ValueError(f"parameter vectors must share one dtype (float32 or float64), got {sorted(map(str, dtypes))}")
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
    elif mode == "delta_sign":
        if w_g_prev is None:
            raise ValueError("delta_sign mode requires w_g_prev")
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
    return RelevanceScore(aligned=int(aligned[0]), total=len(w_c))


def filter_update(update, w_g: ParamVector, w_g_prev: ParamVector | None,
                  policy: SelectionPolicy) -> tuple[bool, RelevanceScore]:
    """Accept iff relevance ratio >= theta (boundary inclusive)."""
    score = calculate_relevance(update.params, w_g, w_g_prev, policy.mode)
    return score.ratio >= policy.theta, score
