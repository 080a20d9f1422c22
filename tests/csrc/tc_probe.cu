// Test-only probe (tests/_tc_probe.so): one CTA computes C[128 x N] = A . B
// with TMA-staged 128B-swizzled operands and tcgen05.mma, for every
// combination of operand majors, using the product's fs_tma.cuh helpers.
// tests/test_gpu_tma_probe.py compares it with torch; it pins the descriptor
// conventions the WIDE trainer relies on.
#include <cuda_bf16.h>
#include <stdio.h>

#include "../../paper_2503_15448_b200/csrc/fs_tma.cuh"

using namespace fs;

template <int N>
__global__ void __launch_bounds__(128) probe_kernel(const __grid_constant__ CUtensorMap ta,
                                                    const __grid_constant__ CUtensorMap tb, int a_mn, int b_mn,
                                                    int K, float* C) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;              // 16 KB
  uint8_t* sb = smem + 16384;      // N * 128 B
  __shared__ uint64_t bar_full, bar_mma;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar_full, 1);
    tc::mbar_init(&bar_mma, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, N < 32 ? 32 : N);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = tc::idesc_bf16(128, N, a_mn != 0, b_mn != 0);
  uint32_t phase = 0;
  for (int k0 = 0; k0 < K; k0 += 64) {
    if (threadIdx.x == 0) {
      tma::expect_tx(&bar_full, 16384u + (uint32_t)N * 128u);
      if (a_mn) {  // A stored [K x 128]: boxes of 64 m-columns x 64 k-rows
        tma::load_3d(sa, &ta, 0, k0, 0, &bar_full);
        tma::load_3d(sa + 8192, &ta, 64, k0, 0, &bar_full);
      } else {     // A stored [128 x K]: one box of 64 k-columns x 128 m-rows
        tma::load_3d(sa, &ta, k0, 0, 0, &bar_full);
      }
      if (b_mn) {  // B stored [K x N]
        for (int j = 0; j < N / 64; ++j) tma::load_3d(sb + j * 8192, &tb, 64 * j, k0, 0, &bar_full);
      } else {     // B stored [N x K]
        tma::load_3d(sb, &tb, k0, 0, 0, &bar_full);
      }
    }
    tc::mbar_wait(&bar_full, phase);
    tc::fence_after_sync();
    if (threadIdx.x == 0) {
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = a_mn ? tma::mnmajor(tc::smem_u32(sa), kk, 8192u) : tma::kmajor(tc::smem_u32(sa), kk);
        const uint64_t bd = b_mn ? tma::mnmajor(tc::smem_u32(sb), kk, 8192u) : tma::kmajor(tc::smem_u32(sb), kk);
        tc::mma_bf16(tmem, ad, bd, idesc, (k0 | kk) != 0);
      }
      tc::mma_commit(&bar_mma);
    }
    tc::mbar_wait(&bar_mma, phase);
    tc::fence_after_sync();
    phase ^= 1;
    __syncthreads();
  }
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
    for (int i = 0; i < 32; ++i) C[(warp * 32 + lane) * N + c0 + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, N < 32 ? 32 : N);
}

extern "C" int probe_gemm(int a_mn, int b_mn, int N, int K, const void* A, const void* B, float* C) {
  CUtensorMap ta, tb;
  bool ok = a_mn ? tma::make_map(&ta, A, 128, K, 1, 128, 0, 64) : tma::make_map(&ta, A, K, 128, 1, K, 0, 128);
  ok = ok && (b_mn ? tma::make_map(&tb, B, N, K, 1, N, 0, 64) : tma::make_map(&tb, B, K, N, 1, K, 0, N));
  if (!ok) return -1;
  const int smem = 1024 + 16384 + N * 128;
  void (*kern)(CUtensorMap, CUtensorMap, int, int, int, float*) = nullptr;
  switch (N) {
    case 64: kern = probe_kernel<64>; break;
    case 128: kern = probe_kernel<128>; break;
    case 256: kern = probe_kernel<256>; break;
    default: return -2;
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<1, 128, smem>>>(ta, tb, a_mn, b_mn, K, C);
  if (cudaDeviceSynchronize() != cudaSuccess) return -3;
  return 0;
}
