"""Per-round evaluation records and metrics.

RoundReport / EvalResult / evaluate mirror pkg/src/fedsim/metrics.py:33-165.
``evaluate`` runs on the device (K8 counts: accuracy at the threshold and
the rank AUC with midrank ties via exact integer 2*U), so the engines never
pull the 43,835 test scores back to the host.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass

import numpy as np

REPORT_SCHEMA_VERSION = 1
ROUND_FIELDS = [
    "schema", "round", "t_s", "accuracy", "auc", "updates", "aggregations", "accepted",
    "rejected", "failures", "accepted_frac", "staleness_mean", "staleness_max",
    "comm_time_s", "transfer_s", "sgd_steps",
]


@dataclass
class EvalResult:
    accuracy: float
    auc: float
    n_pos: int
    n_neg: int
    threshold: float = 0.5


@dataclass
class RoundReport:
    """Per-round record emitted by the engines (metrics.py:92-115)."""

    round: int
    t_s: float
    accuracy: float
    auc: float
    updates: int
    aggregations: int
    accepted: int
    rejected: int
    failures: int
    accepted_frac: float
    staleness_mean: float
    staleness_max: int
    comm_time_s: float
    transfer_s: float
    sgd_steps: int

    def to_record(self) -> dict:
        rec = {"schema": REPORT_SCHEMA_VERSION}
        rec.update(asdict(self))
        return {k: rec[k] for k in ROUND_FIELDS}


def evaluate_device(scores, labels_i8, threshold: float = 0.5) -> EvalResult:
    """K8 metrics on device tensors (scores float64, labels int8)."""
    from . import device as D

    counts = D.eval_counts(scores, labels_i8, threshold).cpu().numpy()
    acc, auc, n_pos, n_neg = D.metrics_from_counts(counts, int(scores.shape[0]))
    return EvalResult(accuracy=acc, auc=auc, n_pos=n_pos, n_neg=n_neg, threshold=threshold)


def evaluate(scores, labels, threshold: float = 0.5) -> EvalResult:
    """Accuracy at ``threshold`` and rank AUC of host or device scores."""
    import torch

    from . import device as D

    rt = D.Runtime.get()
    s = scores if isinstance(scores, torch.Tensor) else rt.h2d(np.asarray(scores, dtype=np.float64))
    lab = labels if isinstance(labels, torch.Tensor) else rt.h2d((np.asarray(labels) == 1).astype(np.int8))
    if s.shape != lab.shape or s.numel() == 0:
        raise ValueError("scores and labels must be equal-length and non-empty")
    return evaluate_device(s.to(torch.float64), lab.to(torch.int8), threshold)


def accuracy(scores, labels, threshold: float = 0.5) -> float:
    return evaluate(scores, labels, threshold).accuracy


def auc_roc(scores, labels) -> float:
    return evaluate(scores, labels).auc


SUMMARY_FIELDS = [
    "schema", "rounds", "accuracy", "auc", "comm_time_s", "transfer_s", "updates", "aggregations",
    "accepted_frac", "staleness_mean", "staleness_max", "sgd_steps", "seed", "mode", "theta",
]


def summarize_reports(reports: list, summary_extra: dict | None = None) -> dict:
    """The one-row run summary (metrics.py:246-275 semantics): last-round
    accuracy/AUC/times, totals over rounds, accepted fraction over decisions."""
    if reports:
        last = reports[-1]
        decided = sum(r.accepted + r.rejected for r in reports)
        summary = {
            "schema": REPORT_SCHEMA_VERSION, "rounds": len(reports), "accuracy": last.accuracy,
            "auc": last.auc, "comm_time_s": last.comm_time_s, "transfer_s": last.transfer_s,
            "updates": sum(r.updates for r in reports), "aggregations": sum(r.aggregations for r in reports),
            "accepted_frac": sum(r.accepted for r in reports) / max(1, decided),
            "staleness_mean": last.staleness_mean,
            "staleness_max": max((r.staleness_max for r in reports), default=0),
            "sgd_steps": sum(r.sgd_steps for r in reports),
        }
    else:
        summary = {"schema": REPORT_SCHEMA_VERSION, "rounds": 0}
    for key in ("seed", "mode", "theta"):
        summary.setdefault(key, "")
    if summary_extra:
        summary.update(summary_extra)
    return summary


def write_reports(reports: list, out_dir: str, summary_extra: dict | None = None) -> dict:
    """rounds.jsonl (one record per report) and summary.csv (header + one
    row; header only for a zero-round run); returns the summary row."""
    import csv
    import json
    import os

    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "rounds.jsonl"), "w", encoding="utf-8") as f:
        for rep in reports:
            f.write(json.dumps(rep.to_record()) + "\n")
    summary = summarize_reports(reports, summary_extra)
    with open(os.path.join(out_dir, "summary.csv"), "w", encoding="utf-8", newline="") as f:
        w = csv.DictWriter(f, fieldnames=SUMMARY_FIELDS, extrasaction="ignore")
        w.writeheader()
        if reports:
            w.writerow({k: summary.get(k, "") for k in SUMMARY_FIELDS})
    return summary
