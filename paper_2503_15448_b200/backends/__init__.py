"""Kernel backend selection — one backend, ``b200``.

Mirrors the reference plugin API (pkg/src/fedsim/backends/__init__.py:1-63):
``get_backend()`` returns a module with NAME, forward, loss_and_grad and
sign_align_count. This framework ships exactly one backend, the sm_100a
C-ABI library; there is no CPU fallback, so FEDSIM_BACKEND accepts only
``auto`` or ``b200`` and the backend fails loudly when its library or GPU
is missing.
"""

from __future__ import annotations

import os

from . import b200

_requested = os.environ.get("FEDSIM_BACKEND", "auto").lower()
if _requested not in ("auto", "b200"):
    raise ImportError(f"FEDSIM_BACKEND must be 'b200' or 'auto' in this framework, got {_requested!r}")

_active = b200


def get_backend():
    """The active kernel module (has forward, loss_and_grad, sign_align_count)."""
    return _active


def backend_name() -> str:
    return _active.NAME


def available_backends() -> list[str]:
    return [b200.NAME]


def unpack_layers(values, dims):
    """Views (no copies) of each layer's (W, b) inside a flat parameter vector
    (reference layout, numpy_backend.py:23-35)."""
    layers = []
    off = 0
    for fan_in, fan_out in zip(dims[:-1], dims[1:]):
        w = values[off : off + fan_in * fan_out].reshape(fan_in, fan_out)
        off += fan_in * fan_out
        b = values[off : off + fan_out]
        off += fan_out
        layers.append((w, b))
    if off != values.shape[0]:
        raise ValueError(f"parameter vector length {values.shape[0]} != layout size {off}")
    return layers
