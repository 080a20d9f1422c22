// Test-only probe (tests/_dmma_probe.so): does the fp64 tensor-core MMA
// (mma.sync.aligned.m8n8k4.row.col.f64) round exactly like a chain of fused
// multiply-adds in k order? The fp64 parity trainer (csrc/fs_train_f64.cu)
// sums every output k = 0..K-1 with one fma per product, which is what keeps
// it bitwise equal to the reference's BLAS; a DMMA inner loop may replace
// that only if the two agree bit for bit (tests/test_gpu_dmma_probe.py).
#include <stdint.h>
#include <string.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// One warp: C[8 x 8] = A[8 x K] . B[K x 8] (row-major A, row-major B),
// out_mma via DMMA over k4 slices, out_fma via a sequential fma chain.
__global__ void dmma_probe_kernel(const double* A, const double* B, int K, double* out_mma,
                                  double* out_fma) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double d0 = 0.0, d1 = 0.0;
  for (int k0 = 0; k0 < K; k0 += 4) {
    const double a = A[g * K + k0 + t];        // A fragment: row g, column t of the k4 slice
    const double b = B[(k0 + t) * 8 + g];      // B fragment: row t of the slice, column g
    dmma(d0, d1, a, b);
  }
  out_mma[g * 8 + 2 * t] = d0;
  out_mma[g * 8 + 2 * t + 1] = d1;
  for (int e = lane; e < 64; e += 32) {
    const int m = e >> 3, n = e & 7;
    double acc = 0.0;
    for (int k = 0; k < K; ++k) acc = fma(A[m * K + k], B[k * 8 + n], acc);
    out_fma[e] = acc;
  }
}

// returns the number of the 64 outputs whose bits differ (-1 on a CUDA error)
extern "C" int probe_dmma(const double* A_host, const double* B_host, int K, double* mma_host,
                          double* fma_host) {
  double *A, *B, *om, *of;
  if (cudaMalloc(&A, sizeof(double) * 8 * K) != cudaSuccess) return -1;
  cudaMalloc(&B, sizeof(double) * 8 * K);
  cudaMalloc(&om, sizeof(double) * 64);
  cudaMalloc(&of, sizeof(double) * 64);
  cudaMemcpy(A, A_host, sizeof(double) * 8 * K, cudaMemcpyHostToDevice);
  cudaMemcpy(B, B_host, sizeof(double) * 8 * K, cudaMemcpyHostToDevice);
  dmma_probe_kernel<<<1, 32>>>(A, B, K, om, of);
  int diff = -1;
  if (cudaDeviceSynchronize() == cudaSuccess) {
    cudaMemcpy(mma_host, om, sizeof(double) * 64, cudaMemcpyDeviceToHost);
    cudaMemcpy(fma_host, of, sizeof(double) * 64, cudaMemcpyDeviceToHost);
    diff = 0;
    for (int i = 0; i < 64; ++i) {
      uint64_t x, y;
      memcpy(&x, mma_host + i, 8);
      memcpy(&y, fma_host + i, 8);
      diff += x != y;
    }
  }
  cudaFree(A);
  cudaFree(B);
  cudaFree(om);
  cudaFree(of);
  return diff;
}
