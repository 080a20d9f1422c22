"""ctypes binding of the C-ABI library ``_fedsim_b200.so`` (include/fedsim_b200.h).

This is the only place the package touches native code. The library is
built in-tree for sm_100a (``paper_2503_15448_b200/csrc/Makefile``) and
there is no fallback: if it is missing, or no CUDA device is visible,
every compute entry point raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_fedsim_b200.so")

FS_OK = 0
FS_EINVAL = -1
FS_ECUDA = -2
FS_ENCCL = -3
FS_EDIVERGED = -4

FS_MASK_NONE = 0
FS_MASK_BITS = 1
FS_MASK_DENSE = 2

FS_OPT_SGD = 0
FS_OPT_ADAM = 1

FS_ALIGN_WEIGHT_SIGN = 0
FS_ALIGN_DELTA_SIGN = 1
FS_COSINE_SCALE = 1 << 40  # fixed-point denominator of delta_cosine scores

FS_MAX_LAYERS = 8

_c_i32 = ctypes.c_int32
_c_i64 = ctypes.c_int64
_c_u64 = ctypes.c_uint64
_c_f64 = ctypes.c_double
_c_vp = ctypes.c_void_p
_c_sz = ctypes.c_size_t


class TrainDesc(ctypes.Structure):
    """Mirror of ``fs_train_desc`` (include/fedsim_b200.h)."""

    _fields_ = [
        ("n_dims", _c_i32),
        ("dims", _c_i32 * (FS_MAX_LAYERS + 1)),
        ("n_req", _c_i32),
        ("epochs", _c_i32),
        ("max_batch", _c_i32),
        ("mask_mode", _c_i32),
        ("scale", _c_f64),
        ("features", _c_vp),
        ("labels", _c_vp),
        ("row_off", _c_vp),
        ("n_rows", _c_vp),
        ("batch", _c_vp),
        ("lr", _c_vp),
        ("w_start", _c_vp),
        ("w_out", _c_vp),
        ("ldw", _c_i64),
        ("perm", _c_vp),
        ("perm_off", _c_vp),
        ("mask_bits", _c_vp),
        ("mask_off", _c_vp),
        ("start_step", _c_vp),
        ("end_step", _c_vp),
        ("order", _c_vp),
        ("status", _c_vp),
        ("workspace", _c_vp),
        ("workspace_bytes", _c_sz),
        ("grid", _c_i32),
        ("mask_flags", _c_vp),
        ("mask_tag", _c_i32),
        ("max_steps", _c_i32),
        ("done", _c_vp),
        ("w_prev", _c_vp),
        ("align_mode", _c_i32),
        ("done_tag", _c_i32),
        ("data_flags", _c_vp),
        ("data_chunk", _c_vp),
        ("data_tag", _c_i32),
        ("align_counts", _c_vp),
        ("w_start_all", _c_vp),
        ("counter_zeroed", _c_i32),
        ("optimizer", _c_i32),
        ("adam_beta1", _c_f64),
        ("adam_beta2", _c_f64),
        ("adam_eps", _c_f64),
        ("opt_state", _c_vp),
        ("max_rows", _c_i32),
    ]


_SIGNATURES = {
    "fs_last_error": (ctypes.c_char_p, []),
    "fs_struct_sizes": (ctypes.c_int32, [_c_vp, _c_i32]),
    "fs_abi_version": (ctypes.c_int, []),
    "fs_memcpy_d2d": (ctypes.c_int, [_c_vp, _c_vp, _c_sz, _c_vp]),
    "fs_fill_u64": (ctypes.c_int, [_c_vp, _c_u64, _c_i64, _c_vp]),
    "fs_publish_flag": (ctypes.c_int, [_c_vp, _c_i32, _c_vp]),
    "fs_upload_chunks": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_vp, _c_i64, _c_vp, _c_i32, _c_vp, _c_i32,
                                        _c_vp]),
    "fs_derive_seed_host": (ctypes.c_int, [_c_u64, ctypes.POINTER(ctypes.c_uint32), _c_i32, ctypes.POINTER(_c_u64)]),
    "fs_train_seeds_host": (ctypes.c_int, [_c_u64, _c_vp, _c_vp, _c_i32, _c_vp]),
    "fs_train_seeds": (ctypes.c_int, [_c_u64, _c_vp, _c_vp, _c_i32, _c_vp, _c_vp]),
    "fs_shuffle_perms": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_i32, _c_i32, _c_i32, _c_vp, _c_vp]),
    "fs_dropout_bits": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp, _c_i32, _c_i32, _c_i32, _c_f64, _c_vp, _c_vp]),
    "fs_dropout_bits_flagged": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_i32, _c_i32, _c_i32, _c_i32,
                                               _c_f64, _c_vp, _c_vp, _c_i32, _c_vp]),
    "fs_dropout_bits_seed": (ctypes.c_int, [_c_u64, _c_i64, _c_f64, _c_vp, _c_vp]),
    "fs_train_workspace_bytes": (_c_sz, [ctypes.POINTER(TrainDesc)]),
    "fs_train_f64": (ctypes.c_int, [ctypes.POINTER(TrainDesc), _c_vp]),
    "fs_bf16_supported": (ctypes.c_int, [_c_vp, _c_i32]),
    "fs_bf16_set_profile": (None, [_c_vp]),
    "fs_bf16_force_generic": (None, [ctypes.c_int]),
    "fs_prep_features_bf16": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_i32, _c_vp, _c_vp, _c_vp]),
    "fs_train_bf16_workspace_bytes": (_c_sz, [ctypes.POINTER(TrainDesc)]),
    "fs_train_bf16": (ctypes.c_int, [ctypes.POINTER(TrainDesc), _c_vp, _c_vp, _c_vp]),
    "fs_step_workspace_bytes": (_c_sz, [_c_vp, _c_i32, _c_i32]),
    "fs_loss_and_grad_f64": (
        ctypes.c_int,
        [_c_vp, _c_i32, _c_vp, _c_vp, _c_vp, _c_i32, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_sz, _c_vp],
    ),
    "fs_forward_workspace_bytes": (_c_sz, [_c_vp, _c_i32, _c_i32]),
    "fs_forward_wide_workspace_bytes": (_c_sz, [_c_vp, _c_i32, _c_i32]),
    "fs_forward_wide": (ctypes.c_int, [_c_vp, _c_i32, _c_vp, _c_vp, _c_i32, _c_vp, _c_vp, _c_sz, _c_vp]),
    "fs_forward_bf16": (ctypes.c_int, [_c_vp, _c_i32, _c_vp, _c_vp, _c_i32, _c_vp, _c_vp]),
    "fs_forward_f64": (ctypes.c_int, [_c_vp, _c_i32, _c_vp, _c_vp, _c_i32, _c_vp, _c_vp, _c_vp, _c_sz, _c_vp]),
    "fs_sign_align_f64": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_i32, _c_i64, _c_i32, _c_vp, _c_vp]),
    "fs_sign_align_f32": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_i32, _c_i64, _c_i32, _c_vp, _c_vp]),
    "fs_sign_align_rows": (ctypes.c_int, [_c_u64, _c_i64, _c_vp, _c_vp, _c_i32, _c_i64, _c_i32, _c_i32, _c_vp, _c_vp]),
    "fs_sign_align_shared": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_i32, _c_i64, _c_i32, _c_i32, _c_vp, _c_vp]),
    "fs_gather_sort_keys_f32": (ctypes.c_int, [_c_vp, _c_i32, _c_i32, _c_vp, _c_vp]),
    "fs_aggregate_f32": (ctypes.c_int, [_c_vp, _c_i32, _c_i64, _c_vp, _c_vp]),
    "fs_gather_sort_keys_f64": (ctypes.c_int, [_c_vp, _c_i32, _c_i32, _c_vp, _c_vp]),
    "fs_canonical_order": (ctypes.c_int, [_c_vp, _c_i32, _c_i64, _c_i32, _c_vp, _c_vp]),
    "fs_aggregate_f64": (ctypes.c_int, [_c_vp, _c_i32, _c_i64, _c_vp, _c_vp]),
    "fs_aggregate_jobs": (ctypes.c_int, [_c_vp, _c_vp, _c_i32, _c_i32, _c_i64, _c_i32, _c_vp, _c_vp, _c_vp]),
    "fs_aggregate_rowsplit_workspace_bytes": (_c_sz, [_c_i64]),
    "fs_aggregate_rowsplit_f32": (ctypes.c_int, [_c_vp, _c_vp, _c_i32, _c_i64, _c_vp, _c_vp, _c_vp, _c_sz, _c_vp]),
    "fs_sum_job": (ctypes.c_int, [_c_vp, _c_vp, _c_i32, _c_i64, _c_i32, _c_vp, _c_vp, _c_vp]),
    "fs_pack_exchange": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_i32, _c_i32, _c_vp, _c_vp, _c_vp]),
    "fs_mean_finish_dev": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_vp, _c_vp, _c_vp]),
    "fs_aggregate_jobs_weighted": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_i32, _c_i32, _c_i64, _c_i32, _c_vp, _c_vp,
                                                  _c_vp, _c_vp]),
    "fs_select_rows": (ctypes.c_int, [_c_vp, _c_i32, _c_i64, _c_f64, _c_i32, _c_i32, _c_u64, _c_i64, _c_vp, _c_vp,
                                      _c_vp, _c_u64, _c_vp]),
    "fs_cosine_align_workspace_bytes": (_c_sz, [_c_i32]),
    "fs_cosine_align": (ctypes.c_int, [_c_vp, _c_u64, _c_i64, _c_vp, _c_vp, _c_i32, _c_i64, _c_i32, _c_vp, _c_vp,
                                       _c_sz, _c_vp]),
    "fs_sum_rows": (ctypes.c_int, [_c_vp, _c_i32, _c_i64, _c_i32, _c_vp, _c_vp]),
    "fs_mean_finish": (ctypes.c_int, [_c_vp, _c_i64, _c_i64, _c_i32, _c_vp, _c_vp]),
    "fs_eval_workspace_bytes": (_c_sz, [_c_i32]),
    "fs_eval_metrics": (ctypes.c_int, [_c_vp, _c_vp, _c_i32, _c_f64, _c_vp, _c_vp, _c_sz, _c_vp]),
    "fs_eval_metrics_f32": (ctypes.c_int, [_c_vp, _c_vp, _c_i32, _c_f64, _c_vp, _c_vp, _c_sz, _c_vp]),
}

# host event engine (bound with its ctypes structs in async_loop.py)
ASYNC_ENGINE_SYMBOLS = ("fs_async_create", "fs_async_destroy", "fs_async_run", "fs_async_provide", "fs_async_log",
                        "fs_async_attach_device")

EXPORTED_SYMBOLS = tuple(_SIGNATURES) + ASYNC_ENGINE_SYMBOLS

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """A CUDA/runtime failure reported by the C-ABI."""


def library_path() -> str:
    return LIB_PATH


def load(require_gpu: bool = True):
    """The loaded C-ABI library; raises if it is not built (no fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"fedsim B200 extension not built: {LIB_PATH} is missing "
                        "(run `make -C paper_2503_15448_b200/csrc` or __graft_entry__.build())"
                    )
                lib = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in _SIGNATURES.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
    if require_gpu:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError(
                "fedsim B200 backend needs a CUDA device; none is visible (no CPU fallback)"
            )
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI status code to the reference's exception types."""
    if rc == FS_OK:
        return
    msg = _lib.fs_last_error().decode(errors="replace") if _lib is not None else ""
    if rc == FS_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise NativeError(f"{what} failed ({rc}): {msg}")
