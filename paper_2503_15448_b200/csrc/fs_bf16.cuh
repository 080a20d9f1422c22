// Shared definitions of the bf16 tensor-core trainers (fs_train_bf16.cu:
// row-major V2 / generic kernels; fs_train_bf16t.cu: unit-major V3 kernel).
#pragma once
#include <cstdio>

#include "fs_common.cuh"
#include "fs_tc.cuh"

namespace fs {
namespace bf16 {

using namespace tc;

constexpr int R = 64;           // batch rows per chunk (MMA M=128; rows >= 64 are ignored)
constexpr int THREADS = 256;    // 8 warps: (lane quarter q = w & 3, column half h = w >> 2)
constexpr int MAXL = 5;         // weight layers supported (<= 4 hidden)
constexpr uint32_t TMEM_COLS = 512;
#ifndef FS_BF16_MAXNREG
// register cap: leaves ~1/3 of the register file for a co-resident kernel
// (the next round's dropout-mask/shuffle prefetch soaks up idle issue slots)
#define FS_BF16_MAXNREG 168
#endif
constexpr int XPRE = 2;         // 16-byte feature chunks per thread per chunk (R * fp0/8 <= 512)

struct Geo {
  int L;
  int f[MAXL + 1];      // true dims
  int fp[MAXL + 1];     // K-padded dims (fp[0] = roundup16(f0); hidden dims already % 16)
  int woff[MAXL], boff[MAXL];
  int M;                // parameters
  int sum_hidden;
  // shared-memory layout (bytes from the dynamic smem base)
  uint32_t s_h[MAXL];   // activation tiles: s_h[0] = X [R x fp0], s_h[l] = H_l [R x f_l]
  uint32_t s_w[MAXL];   // weight tiles W_l [fp_l x f_{l+1}] (hidden layers only)
  uint32_t s_misc;      // fp32 scratch: z, dz, y, zpart[2][R], gw_head, gb
  uint32_t s_bias;      // fp32 copies of the hidden-layer biases (sum_hidden floats)
  int bias_off[MAXL];   // offset of b_l inside s_bias
  uint32_t s_w2m;       // V2: fp32 master of W_2, column-major [f3][f2]
  int v2;               // V2 eligible (3 hidden layers fitting the on-chip optimizer state)
  uint32_t smem_bytes;
};

struct Args {
  Geo g;
  int n_req, epochs, mask_mode;
  float scale;
  const __nv_bfloat16* feat;  // [rows x fp0] bf16, zero padded
  const float* labels;        // [rows]
  const int64_t* row_off;
  const int32_t* n_rows;
  const int32_t* batch;
  const double* lr;           // [n_req x epochs]
  const uint64_t* w_start;    // fp32 flat start parameters
  const float* w_all;         // unit-major kernel: the start model of every request when w_start == nullptr
  float* w_out;               // fp32 flat, ldw floats per request
  int64_t ldw;
  const int32_t* perm;
  const int64_t* perm_off;
  const uint32_t* mask_bits;
  const int64_t* mask_off;
  const int32_t* start_step;
  const int32_t* end_step;
  const int32_t* order;
  int32_t* status;
  int* counter;
  const int32_t* mask_flags;  // per (request, step) readiness of the keep bits (nullptr: complete)
  int32_t mask_tag, max_steps;
  // per-client completion (async engine): after a client's row is written the
  // CTA counts its sign alignment against (w_start, w_prev) and publishes
  // {aligned, status, tag} to done[r] (mapped host memory); nullptr: off
  const uint64_t* done;       // [n_req] device pointers of fs_client_done records
  const uint64_t* w_prev;     // [n_req] previous global (delta_sign) or 0
  int32_t align_mode;         // FS_ALIGN_*, or -1: no count
  int32_t done_tag;
  int64_t* counts_out;        // [n_req] fused K6 counts (sync rounds), nullptr: off
  const int32_t* data_flags;  // chunked shard upload in flight: request r waits on data_flags[data_chunk[r]]
  const int32_t* data_chunk;
  int32_t data_tag;
  float* gacc;                // [grid x M] fp32 gradient accumulators (multi-chunk steps)
  unsigned long long* prof;   // optional [32] phase cycle counters (thread 0 of every CTA)
};

// Phase profiler: thread 0 attributes elapsed SM cycles to phase k.
#define FS_PROF(k)                                        \
  do {                                                    \
    if (a.prof && tid == 0) {                             \
      const long long t1_ = clock64();                    \
      s_prof[k] += (unsigned long long)(t1_ - prof_t0);   \
      prof_t0 = t1_;                                      \
    }                                                     \
  } while (0)

__device__ __forceinline__ float sigmoidf_stable(float z) {
  if (z >= 0.f) return 1.f / (1.f + __expf(-z));
  const float e = __expf(z);
  return e / (1.f + e);
}

__device__ __forceinline__ void stage_sync() {
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
}

__device__ __forceinline__ void wait_mma(uint64_t* bar, uint32_t& phase) {
  mbar_wait(bar, phase);
  phase ^= 1u;
  fence_after_sync();
}


int make_geo(const int32_t* dims, int32_t n_dims, Geo* out);

}  // namespace bf16

// unit-major trainer (fs_train_bf16t.cu): layout check and launch
namespace bf16t {
bool geo_ok(const bf16::Geo& g);
uint32_t smem_bytes(const bf16::Geo& g);
int launch(const bf16::Args& a, int grid, cudaStream_t st);
int launch_eval(const bf16::Geo& g, const float* w, const void* xb, int n, double* probs, cudaStream_t st);
}  // namespace bf16t
}  // namespace fs
