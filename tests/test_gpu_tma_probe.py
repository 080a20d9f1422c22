"""Descriptor conventions of the TMA + tcgen05 kernels (csrc/fs_tma.cuh):
one CTA computes C = A . B from TMA-staged, 128B-swizzled operands for every
combination of K-major / MN-major A and B, against torch (fp32 accumulate of
bf16 inputs). Built by the csrc Makefile as tests/_tc_probe.so."""

import ctypes
import os

import pytest
import torch

from tests.conftest import ROOT, cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

LIB = os.path.join(ROOT, "tests", "_tc_probe.so")


@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("n,k", [(64, 64), (128, 192), (256, 128)])
def test_tma_swizzled_mma_matches_torch(a_mn, b_mn, n, k):
    lib = ctypes.CDLL(LIB)
    g = torch.Generator(device="cuda").manual_seed(7 + n + k)
    a = torch.randn(128, k, device="cuda", generator=g).to(torch.bfloat16)  # logical A [M x K]
    b = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)    # logical B^T [N x K]
    a_store = a.t().contiguous() if a_mn else a.contiguous()                # MN-major: [K x M]
    b_store = b.t().contiguous() if b_mn else b.contiguous()                # MN-major: [K x N]
    c = torch.zeros(128, n, device="cuda", dtype=torch.float32)
    rc = lib.probe_gemm(a_mn, b_mn, n, k, ctypes.c_void_p(a_store.data_ptr()), ctypes.c_void_p(b_store.data_ptr()),
                        ctypes.c_void_p(c.data_ptr()))
    assert rc == 0
    want = a.float() @ b.float().t()
    assert torch.allclose(c, want, rtol=1e-4, atol=1e-3), (c - want).abs().max().item()
