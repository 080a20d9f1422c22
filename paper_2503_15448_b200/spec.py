"""Architecture and batch records of the anomaly MLP (host side).

ModelSpec and Batch keep the reference's fields, digest and validation
(pkg/src/fedsim/model.py:31-122); the parameter container and the
compute entry points live in :mod:`paper_2503_15448_b200.model`.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ModelSpec:
    """MLP architecture: input width, relu hidden widths, one sigmoid unit."""

    input_dim: int
    hidden_dims: tuple[int, ...] = (256, 128, 64)
    output_dim: int = 1
    dropout_rate: float = 0.3
    activation: str = "relu"

    def __post_init__(self):
        hidden = tuple(int(w) for w in self.hidden_dims)
        object.__setattr__(self, "hidden_dims", hidden)
        problems = [
            (self.input_dim >= 1, f"input_dim must be >= 1, got {self.input_dim}"),
            (len(hidden) > 0 and min(hidden) >= 1, f"hidden_dims must be non-empty positive, got {hidden}"),
            (self.output_dim == 1, "only a single sigmoid output unit is supported"),
            (0.0 <= self.dropout_rate < 1.0, f"dropout_rate must be in [0,1), got {self.dropout_rate}"),
            (self.activation == "relu", f"unsupported activation {self.activation!r}"),
        ]
        for ok, why in problems:
            if not ok:
                raise ValueError(why)

    @property
    def dims(self) -> tuple[int, ...]:
        return (self.input_dim,) + self.hidden_dims + (self.output_dim,)

    @property
    def param_count(self) -> int:
        widths = self.dims
        return sum(w_out * (w_in + 1) for w_in, w_out in zip(widths, widths[1:]))

    def digest(self) -> str:
        return _spec_digest(self.input_dim, self.hidden_dims, self.output_dim, self.dropout_rate, self.activation)


_DIGESTS: dict = {}


def _spec_digest(input_dim, hidden, output_dim, rate, activation) -> str:
    key = (input_dim, hidden, output_dim, rate, activation)
    got = _DIGESTS.get(key)
    if got is None:
        payload = json.dumps(
            {"input_dim": input_dim, "hidden_dims": list(hidden), "output_dim": output_dim,
             "dropout_rate": rate, "activation": activation},
            sort_keys=True,
        )
        got = hashlib.blake2b(payload.encode(), digest_size=8).hexdigest()
        _DIGESTS[key] = got
    return got


@dataclass
class Batch:
    """Rows of one SGD step: float64 features [b x d] and 0/1 labels [b]."""

    features: np.ndarray
    labels: np.ndarray

    def __post_init__(self):
        x = np.ascontiguousarray(self.features, dtype=np.float64)
        y = np.ascontiguousarray(self.labels, dtype=np.float64)
        self.features, self.labels = x, y
        if (x.ndim, y.ndim) != (2, 1):
            raise ValueError("features must be 2-D and labels 1-D")
        if len(x) != len(y):
            raise ValueError("features and labels disagree on batch size")
        if len(x) == 0:
            raise ValueError("batch must contain at least one row")
        if not np.isfinite(x).all():
            raise ValueError("batch features contain non-finite values")
        if np.any((y != 0.0) & (y != 1.0)):
            raise ValueError("labels must be 0 or 1")

    @property
    def size(self) -> int:
        return len(self.features)
