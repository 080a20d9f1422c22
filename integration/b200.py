"""B200 kernel backend for the reference ``fedsim`` package.

This is the ONE module a maintainer adds to the reference tree as
``fedsim/backends/b200.py`` (plus the two-line selection hook in
``integration/backends_init.patch``) to run the reference's plugin contract
(pkg/src/fedsim/backends/__init__.py:1-63; numpy_backend.py:3-14;
_core.pyx:93-236) on the sm_100a C-ABI library ``_fedsim_b200.so``:

    NAME, forward(values, dims, x, masks=None),
    loss_and_grad(values, dims, x, y, masks=None), sign_align_count(a, b)

Inputs are borrowed host arrays and outputs fresh float64 numpy arrays, as
with the reference's backends; errors follow them too (ValueError on a
layout or length mismatch). It binds the C ABI with ctypes only: no import
of the B200 framework's Python package. torch is used for device memory and
the current stream. The library is found through ``FEDSIM_B200_LIB`` or by
walking up from this file to ``paper_2503_15448_b200/_fedsim_b200.so``.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

NAME = "b200"

_FS_EINVAL = -1


def _find_lib() -> str:
    path = os.environ.get("FEDSIM_B200_LIB")
    if path:
        return path
    d = os.path.dirname(os.path.abspath(__file__))
    while True:
        cand = os.path.join(d, "paper_2503_15448_b200", "_fedsim_b200.so")
        if os.path.exists(cand):
            return cand
        up = os.path.dirname(d)
        if up == d:
            raise ImportError("fedsim b200 backend: _fedsim_b200.so not found (set FEDSIM_B200_LIB)")
        d = up


if not torch.cuda.is_available():
    raise ImportError("fedsim b200 backend: no CUDA device")
_lib = ctypes.CDLL(_find_lib())
_vp, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
_lib.fs_last_error.restype = ctypes.c_char_p
_lib.fs_step_workspace_bytes.restype = _sz
_lib.fs_step_workspace_bytes.argtypes = [_vp, _i32, _i32]
_lib.fs_forward_workspace_bytes.restype = _sz
_lib.fs_forward_workspace_bytes.argtypes = [_vp, _i32, _i32]
_lib.fs_loss_and_grad_f64.restype = ctypes.c_int
_lib.fs_loss_and_grad_f64.argtypes = [_vp, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
_lib.fs_forward_f64.restype = ctypes.c_int
_lib.fs_forward_f64.argtypes = [_vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _sz, _vp]
_lib.fs_sign_align_f64.restype = ctypes.c_int
_lib.fs_sign_align_f64.argtypes = [_vp, _vp, _vp, _i32, _i64, _i32, _vp, _vp]


def _check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = f"{what}: {_lib.fs_last_error().decode()}"
    if rc == _FS_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _dev(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _layout(values, dims):
    """dims as a C array after the reference's layout check (_core.pyx:93-106)."""
    dims = tuple(int(v) for v in dims)
    size = sum((a + 1) * b for a, b in zip(dims[:-1], dims[1:]))
    n = int(np.shape(values)[0])
    if n != size:
        raise ValueError(f"parameter vector length {n} != layout size {size}")
    return (ctypes.c_int32 * len(dims))(*dims), len(dims), dims


def _masks(masks, rows: int, dims):
    if masks is None:
        return None
    parts = [np.asarray(m, dtype=np.float64).reshape(-1) for m in masks]
    if len(parts) != len(dims) - 2 or any(p.size != rows * h for p, h in zip(parts, dims[1:-1])):
        raise ValueError("one [rows x hidden] dropout mask per hidden layer is required")
    return _dev(np.concatenate(parts)) if parts else None


def forward(values, dims, x, masks=None):
    """Class-1 probabilities for a batch; ``masks=None`` means eval mode (_core.pyx:109-137)."""
    d, nd, dims = _layout(values, dims)
    x = np.asarray(x, dtype=np.float64)
    rows = int(x.shape[0])
    if rows == 0:
        return np.empty(0, dtype=np.float64)
    w, xd, md = _dev(values), _dev(x), _masks(masks, rows, dims)
    probs = torch.empty(rows, dtype=torch.float64, device="cuda")
    ws = torch.empty(max(int(_lib.fs_forward_workspace_bytes(d, nd, rows)), 1), dtype=torch.uint8, device="cuda")
    _check(_lib.fs_forward_f64(d, nd, w.data_ptr(), xd.data_ptr(), rows, None if md is None else md.data_ptr(),
                               probs.data_ptr(), ws.data_ptr(), ws.numel(), _stream()), "forward")
    return probs.cpu().numpy()


def loss_and_grad(values, dims, x, y, masks=None):
    """Mean BCE from logits and its exact flat gradient (_core.pyx:140-219)."""
    d, nd, dims = _layout(values, dims)
    x = np.asarray(x, dtype=np.float64)
    rows = int(x.shape[0])
    w, xd, yd, md = _dev(values), _dev(x), _dev(np.asarray(y).reshape(-1)), _masks(masks, rows, dims)
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    grad = torch.empty_like(w)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = torch.empty(max(int(_lib.fs_step_workspace_bytes(d, nd, rows)), 1), dtype=torch.uint8, device="cuda")
    _check(_lib.fs_loss_and_grad_f64(d, nd, w.data_ptr(), xd.data_ptr(), yd.data_ptr(), rows,
                                     None if md is None else md.data_ptr(), loss.data_ptr(), grad.data_ptr(),
                                     status.data_ptr(), ws.data_ptr(), ws.numel(), _stream()), "loss_and_grad")
    return float(loss.item()), grad.cpu().numpy()


def sign_align_count(a, b):
    """Positions where sign(a) == sign(b), zero its own class (_core.pyx:222-236)."""
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    if a.shape[0] != b.shape[0]:
        raise ValueError("length mismatch")
    if a.shape[0] == 0:
        return 0
    ad, bd = _dev(a), _dev(b)
    ptrs = torch.tensor([ad.data_ptr(), bd.data_ptr()], dtype=torch.int64).to("cuda")
    out = torch.empty(1, dtype=torch.int64, device="cuda")
    _check(_lib.fs_sign_align_f64(ptrs.data_ptr(), ptrs.data_ptr() + 8, None, 1, a.shape[0], 0, out.data_ptr(),
                                  _stream()), "sign_align_count")
    return int(out.item())
