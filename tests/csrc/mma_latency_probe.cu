// Test-only microbenchmark (tests/_mma_latency_probe.so): cycles from the
// first tcgen05.mma issue to the commit's mbarrier completion for one
// "stage" of n_mma MMAs (M = 128, N, K = 16 each) issued by one thread, with
// the operands in the bf16 trainer's SWIZZLE_NONE core-matrix layout or the
// 128-byte-swizzled layout. Diagnoses whether the trainer's per-stage MMA
// time is operand-layout bound or fixed latency.
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../paper_2503_15448_b200/csrc/fs_tc.cuh"
#include "../../paper_2503_15448_b200/csrc/fs_tma.cuh"

using namespace fs;

__device__ __forceinline__ void mma_acc(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
}
__device__ __forceinline__ void mma_first(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
}
template <int NM>
__device__ __forceinline__ void issue_const(uint32_t d, uint64_t ad, uint64_t bd, uint64_t ia, uint64_t ib,
                                            uint32_t idesc) {
  mma_first(d, ad, bd, idesc);
#pragma unroll
  for (int k = 1; k < NM; ++k) mma_acc(d, ad + k * ia, bd + k * ib, idesc);
}

// ~100 KB of straight-line code: run between repetitions it evicts the
// instruction caches, as the bf16 trainer's loop body does between stages
__device__ __noinline__ uint32_t icache_thrash(uint32_t x) {
#pragma unroll
  for (int i = 0; i < 2000; ++i) x = (x ^ (x >> 7)) * (0x9E3779B1u + 2u * (uint32_t)i);
  return x;
}

__global__ void __launch_bounds__(128) mma_lat_kernel(int swz, int N, int n_mma, int nacc, int reps, long long* out) {
  const bool thrash = (swz & 8) != 0;
  swz &= 7;
  uint32_t sink = threadIdx.x;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  // zero operands (values do not matter for timing)
  for (int i = threadIdx.x; i < 128 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&tbase, 512);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t a = tc::smem_u32(smem), b = a + 64 * 1024;
  const uint32_t idesc = tc::idesc_bf16(128, N, false, false);
  uint32_t phase = 0;
  long long total = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (thrash) {
      sink = icache_thrash(sink);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const long long t0 = clock64();
      if (swz == 3) {  // + compile-time count and accumulate flag
        const tc::Tile ta{a, 128}, tb{b, N};
        const uint64_t ad = ta.kmajor(0), bd = tb.kmajor(0);
        const uint64_t ia = ta.kmajor(1) - ad, ib = tb.kmajor(1) - bd;
        if (n_mma == 4) issue_const<4>(tbase, ad, bd, ia, ib, idesc);
        else if (n_mma == 8) issue_const<8>(tbase, ad, bd, ia, ib, idesc);
        else issue_const<16>(tbase, ad, bd, ia, ib, idesc);
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, phase);
        total += clock64() - t0;
      } else if (swz == 2) {  // SWIZZLE_NONE, descriptors advanced by a constant (no per-MMA address math)
        const tc::Tile ta{a, 128}, tb{b, N};
        uint64_t ad = ta.kmajor(0), bd = tb.kmajor(0);
        const uint64_t ia = ta.kmajor(1) - ad, ib = tb.kmajor(1) - bd;
        const uint32_t acc_stride = (uint32_t)N;
#pragma unroll 16
        for (int k = 0; k < n_mma; ++k) {
          tc::mma_bf16(tbase + (nacc > 1 ? (uint32_t)(k & (nacc - 1)) * acc_stride : 0u), ad, bd, idesc, k >= nacc);
          ad += ia;
          bd += ib;
        }
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, phase);
        total += clock64() - t0;
      } else {
      for (int k = 0; k < n_mma; ++k) {
        uint64_t ad, bd;
        if (swz) {  // K-major SW128: K slices within 128-byte rows, 4 per 64-column block
          ad = tma::kmajor(a + (uint32_t)(k / 4) * 128u * 128u, k % 4);
          bd = tma::kmajor(b + (uint32_t)(k / 4) * (uint32_t)N * 128u, k % 4);
        } else {    // SWIZZLE_NONE 8x8 core matrices (fs_tc.cuh Tile::kmajor)
          const tc::Tile ta{a, 128}, tb{b, N};
          ad = ta.kmajor(k);
          bd = tb.kmajor(k);
        }
        tc::mma_bf16(tbase + (uint32_t)((k % nacc) * N), ad, bd, idesc, k >= nacc);
      }
      tc::mma_commit(&bar);
      tc::mbar_wait(&bar, phase);
      total += clock64() - t0;
      }
    }
    phase ^= 1;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = total / reps;
  if (sink == 0x12345678u) out[1] = sink;
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tbase, 512);
}

extern "C" long long probe_mma_latency(int swz, int N, int n_mma, int nacc, int reps) {
  long long* d;
  cudaMalloc(&d, 16);
  const int smem = 1024 + 128 * 1024;
  cudaFuncSetAttribute(mma_lat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_lat_kernel<<<1, 128, smem>>>(swz, N, n_mma, nacc, reps, d);
  long long h = -1;
  if (cudaDeviceSynchronize() == cudaSuccess) cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h;
}
