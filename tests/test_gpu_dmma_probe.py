"""The fp64 parity trainer's GEMMs run on fp64 tensor-core MMA
(mma.sync m8n8k4 f64, csrc/fs_train_f64.cu cta_gemm). That keeps the
reference's rounding only if a DMMA adds its four products in k order with
one rounding each, exactly like a chain of fma() calls; this pins it on the
hardware, including heavy cancellation and mixed magnitudes, bit for bit.
Built by the csrc Makefile as tests/_dmma_probe.so (test-only)."""

import ctypes
import os

import numpy as np
import pytest

from tests.conftest import ROOT, cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

LIB = os.path.join(ROOT, "tests", "_dmma_probe.so")
P = ctypes.POINTER(ctypes.c_double)


def _operands(rng, kind, K):
    if kind == "normal":
        return rng.standard_normal((8, K)), rng.standard_normal((K, 8))
    if kind == "magnitudes":
        return (rng.standard_normal((8, K)) * 10.0 ** rng.integers(-8, 8, (8, K)),
                rng.standard_normal((K, 8)) * 10.0 ** rng.integers(-8, 8, (K, 8)))
    if kind == "cancel":
        a, b = rng.standard_normal((8, K)), rng.standard_normal((K, 8))
        a[:, 1::2] = -a[:, 0::2] * (1 + 1e-13)
        return a, b
    # relu activations x small gradients, with exact zeros (the trainer's dW shape)
    return np.maximum(rng.standard_normal((8, K)), 0) * 3, rng.standard_normal((K, 8)) * 0.05


@pytest.mark.parametrize("kind", ["normal", "magnitudes", "cancel", "relu"])
@pytest.mark.parametrize("K", [4, 44, 256])
def test_dmma_rounds_like_fma_chain(kind, K):
    lib = ctypes.CDLL(LIB)
    rng = np.random.default_rng(K * 7 + len(kind))
    for _ in range(10):
        a, b = (np.ascontiguousarray(x) for x in _operands(rng, kind, K))
        got, want = np.zeros(64), np.zeros(64)
        diff = lib.probe_dmma(a.ctypes.data_as(P), b.ctypes.data_as(P), K, got.ctypes.data_as(P),
                              want.ctypes.data_as(P))
        assert diff == 0, (kind, K, np.abs(got - want).max())
