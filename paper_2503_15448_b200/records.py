"""Client-side records: static profile, finished update, mid-round progress
(fields of pkg/src/fedsim/client.py:29-69)."""

from __future__ import annotations

import math
from dataclasses import dataclass

from .fault import WeibullModel
from .model import ParamVector
from .selection import RelevanceScore


@dataclass
class ClientProfile:
    """Static client characteristics drawn at world build (client.py:29-47)."""

    id: int
    speed: float  # samples processed per simulated second
    up_latency_s: float
    down_latency_s: float
    capacity: float  # resource score driving the batch-size assignment
    dropout_rate: float = 0.0
    weibull: WeibullModel | None = None

    def __post_init__(self):
        if not (math.isfinite(self.speed) and self.speed > 0):
            raise ValueError(f"speed must be positive finite, got {self.speed}")
        if min(self.up_latency_s, self.down_latency_s) < 0:
            raise ValueError("latencies must be >= 0")
        if not self.capacity > 0:
            raise ValueError("capacity must be > 0")
        if not 0.0 <= self.dropout_rate <= 1.0:
            raise ValueError("dropout_rate must be in [0,1]")


@dataclass
class ClientUpdate:
    client_id: int
    round: int
    params: ParamVector
    num_samples: int
    train_time_s: float
    relevance: RelevanceScore | None = None
    steps: int = 0


@dataclass
class TrainingProgress:
    """Mid-round state captured at a batch boundary (checkpoint payload)."""

    params: ParamVector
    epoch: int
    batch_index: int  # next batch to run within the epoch
    steps_done: int
    samples_done: int
