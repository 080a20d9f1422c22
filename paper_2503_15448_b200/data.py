"""Synthetic tabular data and client partitioning for the world build.

One-time host work (out of the hot path). Same streams and arithmetic as
pkg/src/fedsim/data.py:35-282 (synth_anomaly, partition_dirichlet,
stratified_split, scale_columns), so both this framework and the CPU oracle
see byte-identical shards (pinned by tests/golden/world_*.json digests).
CSV ingest is not part of the hot path and is not provided.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .rng import derive_rng


@dataclass
class Dataset:
    features: np.ndarray  # [n x d] float64, scaled
    labels: np.ndarray  # [n] int8 in {0,1}
    feature_names: list
    scaling_stats: tuple

    def __post_init__(self):
        self.features = np.ascontiguousarray(self.features, dtype=np.float64)
        self.labels = np.ascontiguousarray(self.labels, dtype=np.int8)

    @property
    def n(self) -> int:
        return self.features.shape[0]

    @property
    def dim(self) -> int:
        return self.features.shape[1]


@dataclass
class Partition:
    assignments: list


def scale_columns(raw: np.ndarray):
    """Population z-score per column; constant columns keep std 1."""
    mean = raw.mean(axis=0)
    std = raw.std(axis=0)
    std = np.where(std == 0.0, 1.0, std)
    return (raw - mean) / std, (mean, std)


def synth_anomaly(n: int, d: int, anomaly_frac: float, separation: float, seed: int) -> Dataset:
    """Gaussian blobs: normals at 0, anomalies shifted along 1/sqrt(d)."""
    if not 0.0 < anomaly_frac < 1.0:
        raise ValueError(f"anomaly_frac must be in (0,1), got {anomaly_frac}")
    n_anom = max(1, int(np.floor(n * anomaly_frac)))
    if n_anom >= n:
        raise ValueError("anomaly_frac leaves no normal rows")
    n_norm = n - n_anom
    shift = separation * (np.ones(d) / np.sqrt(d))
    normals = derive_rng(seed, "normals").normal(size=(n_norm, d))
    anomalies = derive_rng(seed, "anomalies").normal(size=(n_anom, d)) + shift
    raw = np.vstack([normals, anomalies])
    labels = np.concatenate([np.zeros(n_norm, dtype=np.int8), np.ones(n_anom, dtype=np.int8)])
    order = derive_rng(seed, "shuffle").permutation(n)
    scaled, stats = scale_columns(raw[order])
    return Dataset(scaled, labels[order], [f"f{i}" for i in range(d)], stats)


def partition_dirichlet(ds: Dataset, num_clients: int, alpha: float, seed: int,
                        indices: np.ndarray | None = None, fraction: float = 1.0,
                        max_retries: int = 100) -> Partition:
    """Dirichlet label-skew split; every client gets at least one row."""
    if num_clients < 1:
        raise ValueError("num_clients must be >= 1")
    if alpha <= 0:
        raise ValueError("alpha must be > 0")
    if not 0.0 < fraction <= 1.0:
        raise ValueError("fraction must be in (0,1]")
    pool = np.arange(ds.n) if indices is None else np.asarray(indices)
    rng = derive_rng(seed, "partition")
    if fraction < 1.0:
        pool = rng.permutation(pool)[: max(num_clients, int(round(len(pool) * fraction)))]
    if num_clients == 1:
        return Partition([np.sort(pool)])
    labels = ds.labels[pool]
    classes = np.unique(labels)
    for _ in range(max_retries):
        chunks: list[list[np.ndarray]] = [[] for _ in range(num_clients)]
        for lab in classes:
            rows = rng.permutation(pool[labels == lab])
            props = rng.dirichlet([alpha] * num_clients)
            cuts = (np.cumsum(props) * len(rows)).astype(int)[:-1]
            for c, part in enumerate(np.split(rows, cuts)):
                chunks[c].append(part)
        sizes = [sum(len(p) for p in ch) for ch in chunks]
        if min(sizes) >= 1:
            return Partition([np.sort(np.concatenate(ch).astype(np.int64)) for ch in chunks])
    raise RuntimeError(f"could not give every one of {num_clients} clients a row after {max_retries} draws")


def stratified_split(ds: Dataset, test_frac: float, seed: int):
    """Per-label proportional holdout -> (train_idx, test_idx), both sorted."""
    if not 0.0 < test_frac < 1.0:
        raise ValueError("test_frac must be in (0,1)")
    rng = derive_rng(seed, "split")
    train, test = [], []
    for lab in np.unique(ds.labels):
        rows = rng.permutation(np.flatnonzero(ds.labels == lab))
        k = max(1, int(round(len(rows) * test_frac)))
        test.append(rows[:k])
        train.append(rows[k:])
    return np.sort(np.concatenate(train)), np.sort(np.concatenate(test))
