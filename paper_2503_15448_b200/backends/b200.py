"""The ``b200`` kernel backend: the reference plugin contract on sm_100a kernels.

Contract (pkg/src/fedsim/backends/numpy_backend.py:3-14 and _core.pyx):
flat float64 parameters laid out per layer as W (fan_in x fan_out,
row-major) then b; relu hidden layers with caller-supplied pre-scaled
dropout masks; a single sigmoid unit trained with mean BCE from logits.

Inputs may be numpy arrays (the reference's per-call contract: borrowed,
outputs are fresh numpy arrays) or float64 CUDA tensors (then outputs stay
on the device). Every call runs the same K5/K8 step code the batched
trainer uses (csrc/fs_train_f64.cu), so per-call and batched results agree
bitwise.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _native as N
from .. import device as D

NAME = "b200"


def _layout_size(dims) -> int:
    return sum((a + 1) * b for a, b in zip(dims[:-1], dims[1:]))


def _check_layout(n_values: int, dims) -> None:
    if len(dims) < 3 or len(dims) > N.FS_MAX_LAYERS + 1 or int(dims[-1]) != 1:
        raise ValueError(f"unsupported layer dims {tuple(dims)}")
    size = _layout_size(dims)
    if n_values != size:
        raise ValueError(f"parameter vector length {n_values} != layout size {size}")


def _dev(a, rt) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=rt.device, dtype=torch.float64).contiguous()
    return rt.h2d(np.ascontiguousarray(a, dtype=np.float64))


def _dense_masks(masks, rows: int, dims, rt) -> torch.Tensor | None:
    if masks is None:
        return None
    hidden = dims[1:-1]
    if len(masks) != len(hidden):
        raise ValueError("one mask per hidden layer is required")
    parts = []
    for m, h in zip(masks, hidden):
        t = _dev(m, rt).reshape(-1)
        if t.numel() != rows * h:
            raise ValueError(f"mask shape mismatch: expected {rows}x{h}")
        parts.append(t)
    return torch.cat(parts)


def forward(values, dims, x, masks=None):
    """Class-1 probabilities for a batch; ``masks=None`` means eval mode."""
    rt = D.Runtime.get()
    dims = tuple(int(v) for v in dims)
    host = not isinstance(x, torch.Tensor)
    _check_layout(len(values), dims)
    xd = _dev(x, rt)
    if xd.dim() != 2 or xd.shape[1] != dims[0]:
        raise ValueError(f"x must be [b x {dims[0]}]")
    w = _dev(values, rt)
    dm = _dense_masks(masks, xd.shape[0], dims, rt)
    if xd.shape[0] == 0:
        out = torch.empty(0, dtype=torch.float64, device=rt.device)
    else:
        out = D.forward_probs(dims, w, xd, dm, rt)
    return out.cpu().numpy() if host else out


def loss_and_grad(values, dims, x, y, masks=None):
    """Mean BCE loss and its exact gradient (flat, same layout as values)."""
    rt = D.Runtime.get()
    dims = tuple(int(v) for v in dims)
    host = not isinstance(values, torch.Tensor)
    _check_layout(len(values), dims)
    xd = _dev(x, rt)
    yd = _dev(y, rt).reshape(-1)
    rows = xd.shape[0]
    if xd.dim() != 2 or xd.shape[1] != dims[0] or yd.numel() != rows or rows < 1:
        raise ValueError("x/y shapes do not match the layer dims")
    w = _dev(values, rt)
    dm = _dense_masks(masks, rows, dims, rt)
    loss, grad, status = loss_and_grad_device(dims, w, xd, yd, dm, rt)
    loss_h = float(loss.item())
    return loss_h, (grad.cpu().numpy() if host else grad)


def loss_and_grad_device(dims, w: torch.Tensor, x: torch.Tensor, y: torch.Tensor, dense_masks, rt):
    """Device-resident variant: (loss[1], grad[M], status[1]) tensors."""
    dims_c, nd = D.dims_array(dims)
    rows = x.shape[0]
    M = _layout_size(dims)
    loss = torch.empty(1, dtype=torch.float64, device=rt.device)
    grad = torch.empty(M, dtype=torch.float64, device=rt.device)
    status = torch.zeros(1, dtype=torch.int32, device=rt.device)
    need = rt.lib.fs_step_workspace_bytes(dims_c, nd, rows)
    ws = rt.scratch("step", need)
    rt.call(
        rt.lib.fs_loss_and_grad_f64(
            dims_c, nd, w.data_ptr(), x.data_ptr(), y.data_ptr(), rows,
            None if dense_masks is None else dense_masks.data_ptr(),
            loss.data_ptr(), grad.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(), rt.stream,
        ),
        "fs_loss_and_grad_f64",
    )
    return loss, grad, status


def sign_align_count(a, b) -> int:
    """Number of positions where sign(a) == sign(b); zero is its own class."""
    rt = D.Runtime.get()
    ad = _dev(a, rt).reshape(-1)
    bd = _dev(b, rt).reshape(-1)
    if ad.numel() != bd.numel():
        raise ValueError("length mismatch")
    out = D.align_requests([ad.data_ptr()], [bd.data_ptr()], None, ad.numel(), "weight_sign", rt)
    return int(out.item())
