// K5 (bf16 mode) for MLPs whose hidden layers do not fit the on-chip
// trainers: the WIDE shape of BASELINE configs[4] (42-1024-1024-1024-1024-1)
// and any other layer widths. Same contract as fs_train_bf16
// (client.train_local, client.py:98-172 with bf16 GEMM operands and fp32
// masters): K2 permutations, K3 keep bits, per-epoch learning rates, BCE on
// logits, plain SGD (model.py:189-221, _core.pyx:140-219).
//
// A 1024x1024 layer (2 MB bf16, 4 MB fp32 master) cannot stay on one SM, so
// the clients of a launch train in lockstep: global SGD step t runs step t
// of every client that has one, and every layer product of that step is ONE
// launch of a hand-written tcgen05 kernel over all those clients (grid.z =
// client). Operands are staged by TMA (3-D tensor maps [slot][row][col]
// over the clients' workspace slots, 128-byte swizzle, zero fill past the
// edges) into a 4-deep shared-memory ring; one thread issues
// tcgen05.mma (bf16 x bf16 -> fp32 in TMEM); the elementwise work is the
// epilogue of the same kernel (TMEM -> registers -> global):
//
//   fwd   Z^T[u][r] = sum_k W_l[k][u] H_l[r][k]    A = W_l (MN-major), B = H_l (K-major)
//         -> H_{l+1}[r][u] = relu(Z + b) * keep * scale (bf16); the last
//            hidden layer also leaves per-(row, 32-unit) head-logit partials
//   head  logits, dz, D_H, SGD of the head and of b_{H-1} (CUDA cores)
//   bwd   dH^T[i][r] = sum_j W_l[i][j] D_{l+1}[r][j]  A = W_l (K-major), B = D_{l+1} (K-major)
//         -> D_l = bf16(dH * scale * [H_l > 0]), SGD of b_{l-1}
//   upd   G[i][u] = sum_r H_l[r][i] D_{l+1}[r][u]      A = H_l (MN-major), B = D_{l+1} (MN-major)
//         -> master W_l[i][u] -= lr * G (fp32, in the caller's output row) and
//            its bf16 copy refreshed in the same pass (no separate convert)
//
// Factored mode (SGD, few rows per client: BASELINE configs[4]'s ~21-row
// clients on 1024-wide layers). A client's weights after t steps are its start
// model plus a low-rank sum, W_l = W0_l - sum_t lr_t H_l(t)^T D_{l+1}(t), of
// rank <= its rows so far. Instead of streaming and rewriting every client's
// dense W each step, the trainer keeps W0 (bf16, one copy per distinct start
// model, L2-resident and shared by every client of the launch) and each
// client's history rows H_l(t), D_{l+1}(t) (the step's own activations,
// packed one step after another). A layer product of step t is the shared-W0
// product plus the history term as extra K chunks of the same MMA chain:
//   fwd   Z^T = W0^T H^T + Dhist^T P^T,  P[r][q] = -lr H[r] . Hhist[q]  (gram_kernel)
//   bwd   dH^T = W0 D^T + Hhist^T Q^T,   Q[r][q] = -lr D[r] . Dhist[q]
// and the trained row is written once, at the end: W_l = W0_l - lr Hhist^T
// Dhist (mat_kernel). Same SGD (the history term is exact, rounded in fp32
// instead of through a bf16 copy of W per step); 4 B per parameter per client
// written once instead of 14 B per parameter per client-step.
//
// Units sit on the MMA's M side (128 per tile) and the step's rows on N, so
// one tcgen05.ld row of TMEM is one unit's values across rows and the
// activation stores of a warp are 32 consecutive units (64 B). Per
// client-step the weights are streamed three times (fwd read, bwd read,
// update read-modify-write + bf16 write: 14 B per parameter), so the trainer
// is HBM-bound at the WIDE shape.
#include <cuda_bf16.h>

#include <algorithm>
#include <vector>

#include "fs_common.cuh"
#include "fs_tma.cuh"

namespace fs {
namespace wide {

constexpr int WIDE_GROUP = 256;   // clients per lockstep group (workspace slots)
constexpr int MAXL = FS_MAX_LAYERS;
constexpr int TM = 128;           // units per tile (MMA M)
constexpr int KC = 64;            // K chunk = one 128-byte swizzle row of bf16
constexpr int UN = 256;           // update tile width along fan-out (MMA N)
#ifndef FS_WIDE_STAGES
#define FS_WIDE_STAGES 3
#endif
constexpr int STAGES = FS_WIDE_STAGES;  // fwd/bwd TMA ring depth
constexpr int THREADS = 128;
constexpr int UPD_THREADS_F = 256;         // mat_kernel (the factored mode's weight write)
constexpr uint32_t A_BYTES = TM * KC * 2;  // 16 KB

__host__ __device__ inline int rup(int x, int m) { return (x + m - 1) / m * m; }
// head-logit partials per row: one per 32-unit warp slice of each 128-unit tile
__host__ __device__ __forceinline__ int zparts(int n_last) { return (n_last + TM - 1) / TM * 4; }

struct Geo {
  MlpLayout lay;
  int H;                  // hidden layers
  int dp;                 // X row width (bf16 features padded to 16)
  int rb;                 // activation rows per slot (multiple of nb)
  int nb;                 // rows per fwd/bwd tile = MMA N (multiple of 16, <= 256)
  int rtiles;             // rb / nb
  int ld[MAXL + 1];       // row stride (elements) of the layer-l activations (0: X = dp)
  int ldw[MAXL];          // row stride of the bf16 copy of W_l: roundup8(f_{l+1})
  size_t wb_off[MAXL], x_off, h_off[MAXL + 1], d_off[MAXL + 1], y_off, z_off, bp_off[MAXL + 1];
  size_t slot_bytes;
  // factored mode (fact = 1): activations are history buffers of rha rows
  // (every step's rows packed), P/Q of one layer [rb x ldpq], and the bf16
  // start weights live in version blocks of ver_bytes (wb_off within a block)
  int fact, rha, ldpq;
  size_t pq_off, ver_bytes;
};

constexpr int FACT_MAX_HIST = 512;  // history rows per client (E x rows) the factored mode takes
constexpr int FACT_VERSIONS = 8;    // distinct start models per launch (bf16 version blocks)
constexpr int FACT_GROUP = 512;     // clients per factored lockstep group

// fact_hist > 0: factored geometry for histories of up to fact_hist rows
static bool make(const fs_train_desc* d, Geo* g, int fact_hist = 0) {
  if (make_layout(d->dims, d->n_dims, &g->lay) != FS_OK) return false;
  const MlpLayout& L = g->lay;
  if (L.L < 2 || L.L > MAXL) return false;
  g->H = L.L - 1;
  g->dp = rup(L.f[0], 16);
  const int mb = std::max(16, rup(d->max_batch, 16));
  g->nb = mb <= 256 ? mb : 128;
  g->rb = rup(mb, g->nb);
  g->rtiles = g->rb / g->nb;
  g->ld[0] = g->dp;
  for (int l = 1; l <= g->H; ++l) g->ld[l] = rup(L.f[l], 8);
  g->fact = fact_hist > 0;
  g->rha = g->fact ? rup(fact_hist + g->rb, KC) : g->rb;
  g->ldpq = g->rha;
  size_t s = 0;
  auto take = [&](size_t bytes) {
    s = (s + 255) / 256 * 256;
    const size_t at = s;
    s += bytes;
    return at;
  };
  for (int l = 0; l < g->H; ++l) g->ldw[l] = rup(L.f[l + 1], 8);
  if (g->fact) {  // start weights: one bf16 copy per version block, not per slot
    size_t v = 0;
    for (int l = 0; l < g->H; ++l) {
      v = (v + 255) / 256 * 256;
      g->wb_off[l] = v;
      v += (size_t)L.f[l] * g->ldw[l] * 2;
    }
    g->ver_bytes = (v + 255) / 256 * 256;
  } else {
    for (int l = 0; l < g->H; ++l) g->wb_off[l] = take((size_t)L.f[l] * g->ldw[l] * 2);
    g->ver_bytes = 0;
  }
  g->x_off = take((size_t)g->rha * g->dp * 2);
  for (int l = 1; l <= g->H; ++l) {
    g->h_off[l] = take((size_t)g->rha * g->ld[l] * 2);
    g->d_off[l] = take((size_t)g->rha * g->ld[l] * 2);
    g->bp_off[l] = g->rtiles > 1 ? take((size_t)g->rtiles * L.f[l] * 4) : 0;
  }
  g->h_off[0] = g->x_off;
  g->y_off = take((size_t)g->rb * 4 * 2);  // labels, dz
  g->z_off = take((size_t)g->rb * zparts(L.f[g->H]) * 4);
  g->pq_off = g->fact ? take((size_t)g->rb * g->ldpq * 2) : 0;
  g->slot_bytes = (s + 255) / 256 * 256;
  return true;
}

// per active client of one lockstep step
struct StepRow {
  int req, slot;
  int rows;          // rows of this step (last batch of an epoch may be short)
  int e, s;          // epoch, step within the epoch
  int global_step;
  float lr;
  int off;           // factored: first history row of this step (= history rows before it); else 0
  int wslot;         // factored: version block of the client's start weights
};

// ------------------------------------------------------------------ setup kernels
__global__ void init_master_kernel(const uint64_t* w_start, const int* reqs, int n, int64_t M, float* w_out,
                                   int64_t ldw) {
  const int a = blockIdx.y;
  if (a >= n) return;
  const int r = reqs[a];
  const float* src = reinterpret_cast<const float*>(w_start[r]);
  float* dst = w_out + (int64_t)r * ldw;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const int64_t m4 = M / 4;
    for (int64_t j = t0; j < m4; j += stride)
      reinterpret_cast<float4*>(dst)[j] = __ldcs(reinterpret_cast<const float4*>(src) + j);
    for (int64_t j = m4 * 4 + t0; j < M; j += stride) dst[j] = src[j];
  } else {
    for (int64_t j = t0; j < M; j += stride) dst[j] = src[j];
  }
}

struct ConvArgs {
  MlpLayout lay;
  int H;
  int ldw[MAXL];
  size_t wb_off[MAXL];
  size_t slot_bytes;
  uint8_t* slots;
  const float* w_out;
  int64_t ldw_out;
};

// bf16 copies of every hidden weight matrix of the listed clients (row stride ldw)
__global__ void convert_kernel(ConvArgs c, const StepRow* rows, int n) {
  const int a = blockIdx.y;
  if (a >= n) return;
  const StepRow sr = rows[a];
  const float* m = c.w_out + (int64_t)sr.req * c.ldw_out;
  uint8_t* sb = c.slots + (size_t)sr.slot * c.slot_bytes;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int l = 0; l < c.H; ++l) {
    const int fin = c.lay.f[l], fout = c.lay.f[l + 1];
    const float* src = m + c.lay.woff[l];
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(sb + c.wb_off[l]);
    const int64_t total = (int64_t)fin * fout;
    for (int64_t j = t0; j < total; j += stride) {
      const int64_t i = j / fout, u = j - i * fout;
      dst[i * c.ldw[l] + u] = __float2bfloat16_rn(src[j]);
    }
  }
}

struct StepArgs {
  MlpLayout lay;
  Geo g;
  uint8_t* slots;
  float* w_out;
  int64_t ldw;
  const __nv_bfloat16* feat;
  const float* labels;
  const int64_t* row_off;
  const int32_t* n_rows;
  const int32_t* batch;
  const int32_t* perm;
  const int64_t* perm_off;
  const uint32_t* mask_bits;
  const int64_t* mask_off;
  int mask_mode;
  float scale;
  int32_t* status;
  // opt-in Adam (fs_train_desc.optimizer): moments [n_req][2][ldw] fp32
  int adam;
  float b1, b2, eps;
  float* opt;
  const uint64_t* w_start;    // [n_req] fp32 start rows (factored mode: W0 of the final write)
};

// SGD as the fp32 masters always did, or the opt-in Adam step of parameter
// `idx` of request sr.req at step t = global_step + 1
__device__ __forceinline__ float opt_apply(const StepArgs& a, const StepRow& sr, int64_t idx, float w, float g) {
  if (!a.adam) return w - sr.lr * g;
  float* m = a.opt + (int64_t)sr.req * 2 * a.ldw;
  float* v = m + a.ldw;
  const float t = (float)(sr.global_step + 1);
  const float c1 = 1.f / (1.f - powf(a.b1, t)), c2 = 1.f / (1.f - powf(a.b2, t));
  const float mi = a.b1 * m[idx] + (1.f - a.b1) * g, vi = a.b2 * v[idx] + (1.f - a.b2) * g * g;
  m[idx] = mi;
  v[idx] = vi;
  return w - sr.lr * (mi * c1) / (sqrtf(vi * c2) + a.eps);
}

__device__ __forceinline__ uint8_t* slot_of(const StepArgs& a, int slot) {
  return a.slots + (size_t)slot * a.g.slot_bytes;
}

// X rows of the step (permuted shard rows, bf16, zero padded) and labels
__global__ void gather_kernel(StepArgs a, const StepRow* rows) {
  const StepRow sr = rows[blockIdx.x];
  uint8_t* sb = slot_of(a, sr.slot);
  __nv_bfloat16* x = reinterpret_cast<__nv_bfloat16*>(sb + a.g.x_off) + (int64_t)sr.off * a.g.dp;
  float* y = reinterpret_cast<float*>(sb + a.g.y_off);
  const int n = a.n_rows[sr.req], B = a.batch[sr.req];
  const int32_t* perm = a.perm + a.perm_off[sr.req] + (int64_t)sr.e * n + (int64_t)sr.s * B;
  const int64_t base = a.row_off[sr.req];
  const int cpr = a.g.dp / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < a.g.rb * cpr; i += blockDim.x) {
    const int r = i / cpr, c = i % cpr;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < sr.rows) v = *reinterpret_cast<const uint4*>(a.feat + (base + perm[r]) * a.g.dp + c * 8);
    *reinterpret_cast<uint4*>(x + (int64_t)r * a.g.dp + c * 8) = v;
  }
  for (int r = threadIdx.x; r < a.g.rb; r += blockDim.x) y[r] = r < sr.rows ? a.labels[base + perm[r]] : 0.f;
}

// ------------------------------------------------------------------ tcgen05 tile machinery
struct Ring {
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t done;
  uint32_t tmem;
};

__device__ __forceinline__ uint8_t* smem_base(uint8_t* raw) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
}

__device__ __forceinline__ void ring_init(Ring& R, uint32_t tmem_cols) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&R.full[s], 1);
      tc::mbar_init(&R.empty[s], 1);
    }
    tc::mbar_init(&R.done, 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&R.tmem, tmem_cols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
}

__device__ __forceinline__ void ring_free(Ring& R, uint32_t tmem_cols) {
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(R.tmem, tmem_cols);
}

// One operand phase of a tile's MMA chain: k chunks of A . B from a pair of
// tensor maps. A MN-major (amn): two boxes of 64 units x 64 k at (m0, k) and
// (m0 + 64, k); else one box of 64 k x 128 units at (k, m0). B: one box of
// 64 k x nb rows at (k, brow). aslot / bslot: the maps' 3rd coordinate.
struct Phase {
  const CUtensorMap* ta;
  const CUtensorMap* tb;
  int k;
  bool amn;
  int aslot, bslot, brow;
};

// fwd/bwd/gram main loop: D[128 x nb] (TMEM) = sum over p1's then p2's chunks
__device__ __forceinline__ void mainloop(Ring& R, uint8_t* smem, int m0, int nb, const Phase& p1, const Phase& p2) {
  const uint32_t stage_bytes = A_BYTES + (uint32_t)nb * 128u;
  const int total = p1.k + p2.k;
  // one lane of warp 0 produces (its siblings park at __syncwarp: a spinning
  // sibling would steal the lane's issue slots), warp 1 issues the MMAs
  // converged (a divergent single issuing lane serialises every tcgen05.mma
  // in a per-lane loop)
  if (threadIdx.x == 0) {
    for (int kc = 0; kc < total; ++kc) {
      const bool first = kc < p1.k;
      const Phase& P = first ? p1 : p2;
      const int kl = first ? kc : kc - p1.k;
      const int s = kc % STAGES;
      const uint32_t ph = (uint32_t)(kc / STAGES) & 1u;
      if (kc >= STAGES) tc::mbar_wait(&R.empty[s], ph ^ 1u);
      uint8_t* a = smem + s * stage_bytes;
      uint8_t* b = a + A_BYTES;
      tma::expect_tx(&R.full[s], stage_bytes);
      if (P.amn) {
        tma::load_3d(a, P.ta, m0, kl * KC, P.aslot, &R.full[s]);
        tma::load_3d(a + 8192, P.ta, m0 + 64, kl * KC, P.aslot, &R.full[s]);
      } else {
        tma::load_3d(a, P.ta, kl * KC, m0, P.aslot, &R.full[s]);
      }
      tma::load_3d(b, P.tb, kl * KC, P.brow, P.bslot, &R.full[s]);
    }
  } else if ((threadIdx.x >> 5) == 1) {  // warp 1 issues, converged (mma_bf16_ws: elect.sync)
    const uint32_t id1 = tc::idesc_bf16(TM, nb, p1.amn, false), id2 = tc::idesc_bf16(TM, nb, p2.amn, false);
    for (int kc = 0; kc < total; ++kc) {
      const bool amn = kc < p1.k ? p1.amn : p2.amn;
      const uint32_t idesc = kc < p1.k ? id1 : id2;
      const int s = kc % STAGES;
      const uint32_t ph = (uint32_t)(kc / STAGES) & 1u;
      tc::mbar_wait(&R.full[s], ph);
      tc::fence_after_sync();
      const uint32_t a = tc::smem_u32(smem + s * stage_bytes), b = a + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < KC / 16; ++kk) {
        const uint64_t ad = amn ? tma::mnmajor(a, kk, 8192u) : tma::kmajor(a, kk);
        tc::mma_bf16_ws(R.tmem, ad, tma::kmajor(b, kk), idesc, (kc | kk) != 0);
      }
      tc::mma_commit_ws(&R.empty[s]);
    }
    tc::mma_commit_ws(&R.done);
  }
  __syncwarp();
  tc::mbar_wait(&R.done, 0);
  tc::fence_after_sync();
}

__device__ __forceinline__ uint32_t lane_addr(uint32_t tmem, int col) {
  return tmem + ((uint32_t)(((threadIdx.x >> 5) & 3) * 32) << 16) + (uint32_t)col;
}

// 32x32 bit transpose across a warp: in, lane k bit u = A[k][u]; out, lane u bit k
__device__ __forceinline__ uint32_t bit_transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int j = 16; j >= 1; j >>= 1) {
    const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu : j == 2 ? 0x33333333u
                                                                                                     : 0x55555555u;
    const uint32_t t = __shfl_xor_sync(0xFFFFFFFFu, x, j);
    x = (lane & j) ? ((x & ~m) | ((t >> j) & m)) : ((x & m) | ((t << j) & ~m));
  }
  return x;
}

// warp reduce-scatter: lane L returns the sum over lanes of p[L] (p clobbered)
__device__ __forceinline__ float reduce_scatter32(float (&p)[32], int lane) {
#pragma unroll
  for (int j = 16; j >= 1; j >>= 1) {
    const bool up = (lane & j) != 0;
#pragma unroll
    for (int i = 0; i < j; ++i) {
      const float send = up ? p[i] : p[i + j];
      const float keep = up ? p[i + j] : p[i];
      p[i] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, j);
    }
  }
  return p[0];
}

// keep bits of rows [rbase, rbase+32) for this warp's 32 units [ub, ub+32):
// lane l fetches the 32 unit bits of row rbase+l (K3 layout: row-major
// [rows x f_l] per hidden layer), a bit transpose hands lane u its row bits
__device__ __forceinline__ uint32_t keep_word(const StepArgs& a, const StepRow& sr, int l, int64_t hid_base,
                                              int rbase, int ub, int lane) {
  const int r = rbase + lane;
  uint32_t w = 0;
  if (r < sr.rows && ub < a.lay.f[l]) {
    const int B = a.batch[sr.req];
    const int64_t slot_words = ((int64_t)B * a.lay.sum_hidden + 31) / 32;
    const uint32_t* bits = a.mask_bits + a.mask_off[sr.req] + (int64_t)sr.global_step * slot_words;
    const int64_t j = (int64_t)sr.rows * hid_base + (int64_t)r * a.lay.f[l] + ub;
    const int64_t last = j + min(32, a.lay.f[l] - ub) - 1;
    const uint32_t sh = (uint32_t)(j & 31);
    w = bits[j >> 5] >> sh;
    if ((last >> 5) != (j >> 5)) w |= bits[(j >> 5) + 1] << (32u - sh);
  }
  return bit_transpose32(w, lane);
}

// ------------------------------------------------------------------ forward
struct FwdArgs {
  int l;              // output layer (1..H): H_l = relu(H_{l-1} W_{l-1} + b_{l-1})
  int fin, fout, nb, kchunks, last, zp;
  int64_t boff, whoff, hid_base;
  // training: per-client slots
  size_t h_off, z_off;
  int ld_out;
  // evaluation (eval = 1): one model, global buffers
  int eval, rows_eval;
  __nv_bfloat16* h_eval;
  float* z_eval;
  const float* w_eval;
};

// factored mode: ta2 = Dhist_{l} [q][u] (MN-major), tb2 = P [r][q] (the history term)
__global__ void __launch_bounds__(THREADS) fwd_kernel(const __grid_constant__ CUtensorMap ta,
                                                      const __grid_constant__ CUtensorMap tb,
                                                      const __grid_constant__ CUtensorMap ta2,
                                                      const __grid_constant__ CUtensorMap tb2, StepArgs a, FwdArgs f,
                                                      const StepRow* rows) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Ring R;
  uint8_t* smem = smem_base(smem_raw);
  const int tile = blockIdx.x, m0 = tile * TM, r0 = blockIdx.y * f.nb;
  StepRow sr{};
  int slot = 0, nrows;
  const float* W;
  if (f.eval) {
    nrows = f.rows_eval;
    W = f.w_eval;
  } else {
    sr = rows[blockIdx.z];
    slot = sr.slot;
    nrows = sr.rows;
    W = a.w_out + (int64_t)sr.req * a.ldw;
  }
  if (threadIdx.x == 0) {
    tma::prefetch_map(&ta);
    tma::prefetch_map(&tb);
  }
  const uint32_t cols = f.nb <= 32 ? 32 : f.nb <= 64 ? 64 : f.nb <= 128 ? 128 : 256;
  ring_init(R, cols);
  {
    const bool fact = !f.eval && a.g.fact;
    const Phase p1{&ta, &tb, f.kchunks, true, fact ? sr.wslot : slot, slot, r0 + sr.off};
    const Phase p2{&ta2, &tb2, fact ? (sr.off + KC - 1) / KC : 0, true, slot, slot, r0};
    mainloop(R, smem, m0, f.nb, p1, p2);
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = m0 + threadIdx.x;
  const bool uok = u < f.fout;
  const float b = uok ? W[f.boff + u] : 0.f;
  const float wh = f.last && uok ? W[f.whoff + u] : 0.f;
  const bool masked = !f.eval && a.mask_mode == FS_MASK_BITS;
  const float sc = masked ? a.scale : 1.f;
  __nv_bfloat16* h = f.eval ? f.h_eval : reinterpret_cast<__nv_bfloat16*>(slot_of(a, slot) + f.h_off);
  float* z = f.eval ? f.z_eval : reinterpret_cast<float*>(slot_of(a, slot) + f.z_off);
  const int rend = f.eval ? min(r0 + f.nb, nrows) : r0 + f.nb;  // training slots hold rb rows
  for (int c0 = 0; c0 < f.nb; c0 += 32) {
    if (r0 + c0 >= rend) break;
    const uint32_t keep = masked ? keep_word(a, sr, f.l, f.hid_base, r0 + c0, m0 + warp * 32, lane) : ~0u;
    float v[32];
    tc::tmem_ld32(lane_addr(R.tmem, c0), v);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int r = r0 + c0 + j;
      float x = 0.f;
      if (r < nrows && uok) {
        x = fmaxf(v[j] + b, 0.f);
        x = ((keep >> j) & 1u) ? x * sc : 0.f;
      }
      if (uok && r < rend && c0 + j < f.nb) h[(int64_t)(sr.off + r) * f.ld_out + u] = __float2bfloat16_rn(x);
      v[j] = x * wh;
    }
    if (f.last) {  // head-logit partial of row r0+c0+lane over this warp's 32 units
      const float p = reduce_scatter32(v, lane);
      const int r = r0 + c0 + lane;
      if (r < nrows && r < rend && c0 + lane < f.nb) z[(int64_t)r * f.zp + tile * 4 + warp] = p;
    }
  }
  ring_free(R, cols);
}

// ------------------------------------------------------------------ head (CUDA cores)
// logits from the fixed-order partials, dz, D_H, SGD on the head and b_{H-1}
__global__ void __launch_bounds__(256) head_kernel(StepArgs a, const StepRow* rows) {
  const StepRow sr = rows[blockIdx.x];
  const int H = a.g.H, N = a.lay.f[H], ld = a.g.ld[H], rb = a.g.rb;
  uint8_t* sb = slot_of(a, sr.slot);
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(sb + a.g.h_off[H]) + (int64_t)sr.off * ld;
  __nv_bfloat16* dout = reinterpret_cast<__nv_bfloat16*>(sb + a.g.d_off[H]) + (int64_t)sr.off * ld;
  const float* y = reinterpret_cast<const float*>(sb + a.g.y_off);
  float* dz = reinterpret_cast<float*>(sb + a.g.y_off) + rb;
  float* W = a.w_out + (int64_t)sr.req * a.ldw;
  float* wh = W + a.lay.woff[H];
  float* bh = W + a.lay.boff[H];
  float* bprev = W + a.lay.boff[H - 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  extern __shared__ float s_dz[];
  __shared__ float s_red[8];
  const float* zacc = reinterpret_cast<const float*>(sb + a.g.z_off);
  const int zp = zparts(N);
  for (int r = threadIdx.x; r < rb; r += blockDim.x) {
    float d = 0.f;
    if (r < sr.rows) {
      float zs = 0.f;
      for (int k = 0; k < zp; ++k) zs += zacc[(int64_t)r * zp + k];
      const float z = zs + bh[0];
      const float sg = z >= 0.f ? 1.f / (1.f + __expf(-z)) : __expf(z) / (1.f + __expf(z));
      d = (sg - y[r]) / (float)sr.rows;
      if (!isfinite(z)) atomicOr(a.status + sr.req, 1);
    }
    s_dz[r] = d;
    dz[r] = d;
  }
  __syncthreads();
  const float sc = a.mask_mode == FS_MASK_BITS ? a.scale : 1.f;
  // a thread takes unit pairs (bf16x2 row accesses); H and D are different
  // buffers (__restrict__), so the row loads of a pair are issued ahead of
  // its D stores instead of one L2 round trip per row (the same products and
  // sums in the same row order as one unit at a time)
  const int npair = (N % 2 == 0 && ld % 2 == 0) ? N / 2 : 0;
  const __nv_bfloat162* __restrict__ h2 = reinterpret_cast<const __nv_bfloat162*>(h);
  __nv_bfloat162* __restrict__ d2 = reinterpret_cast<__nv_bfloat162*>(dout);
  auto update = [&](int u, float w, float g, float gb) {
    if (a.adam) {
      wh[u] = opt_apply(a, sr, a.lay.woff[H] + u, w, g);
      bprev[u] = opt_apply(a, sr, a.lay.boff[H - 1] + u, bprev[u], gb);
    } else {
      wh[u] = w - sr.lr * g;
      bprev[u] -= sr.lr * gb;
    }
  };
  for (int up = threadIdx.x; up < npair; up += blockDim.x) {
    const float w0 = wh[2 * up], w1 = wh[2 * up + 1];
    float g0 = 0.f, g1 = 0.f, gb0 = 0.f, gb1 = 0.f;
#pragma unroll 8
    for (int r = 0; r < rb; ++r) {
      const float2 hv = __bfloat1622float2(h2[(int64_t)r * (ld / 2) + up]);
      const float dzr = s_dz[r];
      g0 = fmaf(hv.x, dzr, g0);
      g1 = fmaf(hv.y, dzr, g1);
      const __nv_bfloat162 dv = __floats2bfloat162_rn(hv.x > 0.f ? dzr * w0 * sc : 0.f, hv.y > 0.f ? dzr * w1 * sc : 0.f);
      d2[(int64_t)r * (ld / 2) + up] = dv;
      const float2 df = __bfloat1622float2(dv);
      gb0 += df.x;
      gb1 += df.y;
    }
    update(2 * up, w0, g0, gb0);
    update(2 * up + 1, w1, g1, gb1);
  }
  for (int u = 2 * npair + threadIdx.x; u < N; u += blockDim.x) {
    const float w = wh[u];
    float g = 0.f, gb = 0.f;
    for (int r = 0; r < rb; ++r) {
      const float hv = __bfloat162float(h[(int64_t)r * ld + u]);
      g = fmaf(hv, s_dz[r], g);
      const __nv_bfloat16 dv = __float2bfloat16_rn(hv > 0.f ? s_dz[r] * w * sc : 0.f);
      dout[(int64_t)r * ld + u] = dv;
      gb += __bfloat162float(dv);
    }
    update(u, w, g, gb);
  }
  float t = 0.f;
  for (int r = threadIdx.x; r < rb; r += blockDim.x) t += s_dz[r];
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) s_red[warp] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w2 = 0; w2 < 8; ++w2) s += s_red[w2];
    if (a.adam) bh[0] = opt_apply(a, sr, a.lay.boff[H], bh[0], s);
    else bh[0] -= sr.lr * s;
  }
}

// ------------------------------------------------------------------ backward
struct BwdArgs {
  int l;              // D_l from D_{l+1} through W_l (1 <= l < H)
  int fin, fout, nb, kchunks;
  int64_t boff;       // b_{l-1}
  size_t h_off, d_off, bp_off;
  int ld;
};

// factored mode: ta2 = Hhist_l [q][i] (MN-major), tb2 = Q [r][q] (the history term)
__global__ void __launch_bounds__(THREADS) bwd_kernel(const __grid_constant__ CUtensorMap ta,
                                                      const __grid_constant__ CUtensorMap tb,
                                                      const __grid_constant__ CUtensorMap ta2,
                                                      const __grid_constant__ CUtensorMap tb2, StepArgs a, BwdArgs p,
                                                      const StepRow* rows) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Ring R;
  uint8_t* smem = smem_base(smem_raw);
  const StepRow sr = rows[blockIdx.z];
  const int m0 = blockIdx.x * TM, r0 = blockIdx.y * p.nb;
  if (threadIdx.x == 0) {
    tma::prefetch_map(&ta);
    tma::prefetch_map(&tb);
  }
  const uint32_t cols = p.nb <= 32 ? 32 : p.nb <= 64 ? 64 : p.nb <= 128 ? 128 : 256;
  ring_init(R, cols);
  {
    const bool fact = a.g.fact;
    const Phase p1{&ta, &tb, p.kchunks, false, fact ? sr.wslot : sr.slot, sr.slot, r0 + sr.off};
    const Phase p2{&ta2, &tb2, fact ? (sr.off + KC - 1) / KC : 0, true, sr.slot, sr.slot, r0};
    mainloop(R, smem, m0, p.nb, p1, p2);
  }

  const int i = m0 + threadIdx.x;
  const bool iok = i < p.fin;
  uint8_t* sb = slot_of(a, sr.slot);
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(sb + p.h_off) + (int64_t)sr.off * p.ld;
  __nv_bfloat16* dl = reinterpret_cast<__nv_bfloat16*>(sb + p.d_off) + (int64_t)sr.off * p.ld;
  const float sc = a.mask_mode == FS_MASK_BITS ? a.scale : 1.f;
  float gb = 0.f;
  for (int c0 = 0; c0 < p.nb; c0 += 32) {
    float v[32];
    tc::tmem_ld32(lane_addr(R.tmem, c0), v);
    if (iok) {
      // every H load of the chunk before the first D store (they may alias)
      __nv_bfloat16 hv[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        hv[j] = c0 + j < p.nb ? h[(int64_t)(r0 + c0 + j) * p.ld + i] : __float2bfloat16_rn(0.f);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (c0 + j >= p.nb) continue;  // nb % 32 == 16: the last chunk is half wide
        const __nv_bfloat16 dv = __float2bfloat16_rn(__bfloat162float(hv[j]) > 0.f ? v[j] * sc : 0.f);
        dl[(int64_t)(r0 + c0 + j) * p.ld + i] = dv;
        gb += __bfloat162float(dv);
      }
    }
  }
  if (iok) {
    if (a.g.rtiles == 1) {
      float* b = a.w_out + (int64_t)sr.req * a.ldw + p.boff + i;
      if (a.adam) *b = opt_apply(a, sr, p.boff + i, *b, gb);
      else *b -= sr.lr * gb;
    }
    else reinterpret_cast<float*>(sb + p.bp_off)[(int64_t)blockIdx.y * p.fin + i] = gb;
  }
  ring_free(R, cols);
}

// b_{l-1} SGD from the per-row-tile partial sums (row tiles > 1), in tile order
__global__ void bias_reduce_kernel(StepArgs a, const StepRow* rows, int fin, int64_t boff, size_t bp_off) {
  const StepRow sr = rows[blockIdx.y];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= fin) return;
  const float* bp = reinterpret_cast<const float*>(slot_of(a, sr.slot) + bp_off);
  float gb = 0.f;
  for (int t = 0; t < a.g.rtiles; ++t) gb += bp[(int64_t)t * fin + i];
  float* b = a.w_out + (int64_t)sr.req * a.ldw + boff + i;
  if (a.adam) *b = opt_apply(a, sr, boff + i, *b, gb);
  else *b -= sr.lr * gb;
}

// ------------------------------------------------------------------ factored mode
// P[r][q] = -lr * sum_k A[q][k] cur[r][k] for the history rows q < sr.off of
// this client (0 beyond), bf16, the B operand of the next fwd/bwd's history
// phase: A = Hhist_l (fwd) or Dhist_{l+1} (bwd), K-major; cur = this step's
// rows of the same buffer (at sr.off). TMEM lane = q, columns = rows.
struct GramArgs {
  int kchunks, nb;
  size_t pq_off;
  int ldpq;
};

__global__ void __launch_bounds__(THREADS) gram_kernel(const __grid_constant__ CUtensorMap ta,
                                                       const __grid_constant__ CUtensorMap tb, StepArgs a, GramArgs p,
                                                       const StepRow* rows) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Ring R;
  uint8_t* smem = smem_base(smem_raw);
  const StepRow sr = rows[blockIdx.z];
  const int q0 = blockIdx.x * TM, r0 = blockIdx.y * p.nb;
  if (q0 >= sr.off) return;  // this client has no history rows in the tile (uniform per CTA)
  if (threadIdx.x == 0) {
    tma::prefetch_map(&ta);
    tma::prefetch_map(&tb);
  }
  const uint32_t cols = p.nb <= 32 ? 32 : p.nb <= 64 ? 64 : p.nb <= 128 ? 128 : 256;
  ring_init(R, cols);
  const Phase p1{&ta, &tb, p.kchunks, false, sr.slot, sr.slot, r0 + sr.off};
  const Phase none{&ta, &tb, 0, false, 0, 0, 0};
  mainloop(R, smem, q0, p.nb, p1, none);
  const int q = q0 + threadIdx.x;
  const float nlr = q < sr.off ? -sr.lr : 0.f;
  __nv_bfloat16* P = reinterpret_cast<__nv_bfloat16*>(slot_of(a, sr.slot) + p.pq_off);
  for (int c0 = 0; c0 < p.nb; c0 += 32) {
    float v[32];
    tc::tmem_ld32(lane_addr(R.tmem, c0), v);
    if (q < p.ldpq) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (c0 + j < p.nb) P[(int64_t)(r0 + c0 + j) * p.ldpq + q] = __float2bfloat16_rn(nlr * v[j]);
    }
  }
  ring_free(R, cols);
}

// the factored trainer's only write of the weights: W_l[i][u] = W0_l[i][u]
// - lr * sum_q Hhist_l[q][i] Dhist_{l+1}[q][u] over the client's sr.off
// history rows (A = Hhist MN-major, B = Dhist MN-major, as upd_kernel)
struct MatArgs {
  int fin, fout;
  int64_t woff;
};

// 128-wide fan-out tiles (64 KB ring, 128 TMEM columns): three CTAs per SM
// keep the write stream going while other CTAs run their (short) main loops
constexpr int UNF = 128;
__global__ void __launch_bounds__(UPD_THREADS_F) mat_kernel(const __grid_constant__ CUtensorMap ta,
                                                            const __grid_constant__ CUtensorMap tb, StepArgs a,
                                                            MatArgs p, const StepRow* rows) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Ring R;
  uint8_t* smem = smem_base(smem_raw);
  const StepRow sr = rows[blockIdx.z];
  const int i0 = blockIdx.x * TM, u0 = blockIdx.y * UNF;
  const int nu = min(UNF, p.fout - u0);
  const int nmma = rup(nu, 16), nbox = (nu + 63) / 64;
  const int kchunks = max(1, (sr.off + KC - 1) / KC);
  const uint32_t stage_bytes = A_BYTES + (uint32_t)nbox * 8192u;
  if (threadIdx.x == 0) {
    tma::prefetch_map(&ta);
    tma::prefetch_map(&tb);
  }
  ring_init(R, UNF);
  if (threadIdx.x == 0) {
    for (int kc = 0; kc < kchunks; ++kc) {
      const int s = kc % 2;
      const uint32_t ph = (uint32_t)(kc / 2) & 1u;
      if (kc >= 2) tc::mbar_wait(&R.empty[s], ph ^ 1u);
      uint8_t* A = smem + s * (A_BYTES + (UNF / 64) * 8192);
      uint8_t* B = A + A_BYTES;
      tma::expect_tx(&R.full[s], stage_bytes);
      tma::load_3d(A, &ta, i0, kc * KC, sr.slot, &R.full[s]);
      tma::load_3d(A + 8192, &ta, i0 + 64, kc * KC, sr.slot, &R.full[s]);
      for (int j = 0; j < nbox; ++j) tma::load_3d(B + j * 8192, &tb, u0 + 64 * j, kc * KC, sr.slot, &R.full[s]);
    }
  } else if ((threadIdx.x >> 5) == 1) {  // warp 1 issues, converged (mma_bf16_ws: elect.sync)
    const uint32_t idesc = tc::idesc_bf16(TM, nmma, true, true);
    for (int kc = 0; kc < kchunks; ++kc) {
      const int s = kc % 2;
      const uint32_t ph = (uint32_t)(kc / 2) & 1u;
      tc::mbar_wait(&R.full[s], ph);
      tc::fence_after_sync();
      const uint32_t A = tc::smem_u32(smem + s * (A_BYTES + (UNF / 64) * 8192)), B = A + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < KC / 16; ++kk)
        tc::mma_bf16_ws(R.tmem, tma::mnmajor(A, kk, 8192u), tma::mnmajor(B, kk, 8192u), idesc, (kc | kk) != 0);
      tc::mma_commit_ws(&R.empty[s]);
    }
    tc::mma_commit_ws(&R.done);
  }
  __syncwarp();
  tc::mbar_wait(&R.done, 0);
  tc::fence_after_sync();

  // epilogue as upd_kernel's: TMEM -> registers -> shared transpose -> whole
  // 128-byte row segments; W0 (the shared start row, L2) read, W written once
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = warp & 3;
  const int nchunk = (nmma + 31) / 32;
  const float nlr = -sr.lr;
  float* T = reinterpret_cast<float*>(smem) + warp * (32 * 36);
  const int rr0 = lane >> 3, cc = (lane & 7) * 4;
  const int64_t base = p.woff + (int64_t)(i0 + q * 32) * p.fout + u0;
  float* wbase = a.w_out + (int64_t)sr.req * a.ldw + base;
  const float* w0 = reinterpret_cast<const float*>(a.w_start[sr.req]) + base;
  const bool vec = (p.fout % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.w_out + p.woff) & 15) == 0) &&
                   ((a.ldw & 3) == 0) && ((reinterpret_cast<uintptr_t>(w0 - base + p.woff) & 15) == 0);
  auto row_ok = [&](int pp) { return i0 + q * 32 + 4 * pp + rr0 < p.fin; };
  for (int c = warp >> 2; c < nchunk; c += 2) {
    float g[32];
    tc::tmem_ld32(lane_addr(R.tmem, 32 * c), g);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      *reinterpret_cast<float4*>(T + lane * 36 + 4 * k) = make_float4(g[4 * k], g[4 * k + 1], g[4 * k + 2], g[4 * k + 3]);
    __syncwarp();
#pragma unroll
    for (int pp = 0; pp < 8; ++pp) {
      if (!row_ok(pp)) continue;
      const int row = 4 * pp + rr0;
      if (vec && 32 * c + cc + 4 <= nu) {
        const float4 g4 = *reinterpret_cast<const float4*>(T + row * 36 + cc);
        float4 w = __ldg(reinterpret_cast<const float4*>(w0 + (int64_t)row * p.fout + 32 * c + cc));
        w.x = fmaf(nlr, g4.x, w.x);
        w.y = fmaf(nlr, g4.y, w.y);
        w.z = fmaf(nlr, g4.z, w.z);
        w.w = fmaf(nlr, g4.w, w.w);
        __stcs(reinterpret_cast<float4*>(wbase + (int64_t)row * p.fout + 32 * c + cc), w);
      } else {
        for (int e = 0; e < 4; ++e) {
          const int u = 32 * c + cc + e;
          if (u >= nu) break;
          wbase[(int64_t)row * p.fout + u] = fmaf(nlr, T[row * 36 + cc + e], w0[(int64_t)row * p.fout + u]);
        }
      }
    }
    __syncwarp();
  }
  ring_free(R, UNF);
}

// biases and head of every listed request from its start row (factored
// mode: the weight blocks are written by mat_kernel at the end)
__global__ void init_small_kernel(const uint64_t* w_start, const int* reqs, int n, MlpLayout L, float* w_out,
                                  int64_t ldw) {
  const int a = blockIdx.y;
  if (a >= n) return;
  const int r = reqs[a];
  const float* src = reinterpret_cast<const float*>(w_start[r]);
  float* dst = w_out + (int64_t)r * ldw;
  for (int l = 0; l < L.L; ++l) {
    const int64_t b0 = L.boff[l], nb = L.f[l + 1];
    for (int64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x)
      dst[b0 + j] = src[b0 + j];
  }
  const int H = L.L - 1;  // head weights [f_H]
  for (int64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < L.f[H]; j += (int64_t)gridDim.x * blockDim.x)
    dst[L.woff[H] + j] = src[L.woff[H] + j];
}

// bf16 copy of the hidden weight matrices of each distinct start model
struct VerArgs {
  MlpLayout lay;
  int H;
  int ldw[MAXL];
  size_t wb_off[MAXL];
  size_t ver_bytes;
  uint8_t* vers;
  const uint64_t* src;  // [nver] fp32 start rows
};

__global__ void version_convert_kernel(VerArgs c) {
  const float* m = reinterpret_cast<const float*>(c.src[blockIdx.y]);
  uint8_t* vb = c.vers + (size_t)blockIdx.y * c.ver_bytes;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int l = 0; l < c.H; ++l) {
    const int fin = c.lay.f[l], fout = c.lay.f[l + 1];
    const float* src = m + c.lay.woff[l];
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(vb + c.wb_off[l]);
    const int64_t total = (int64_t)fin * fout;
    for (int64_t j = t0; j < total; j += stride) {
      const int64_t i = j / fout, u = j - i * fout;
      dst[i * c.ldw[l] + u] = __float2bfloat16_rn(src[j]);
    }
  }
}

// ------------------------------------------------------------------ update
struct UpdArgs {
  int l;              // W_l [fin x fout] from H_l and D_{l+1}
  int fin, fout;
  int64_t woff;
  size_t wb_off;
  int ldw;
};

constexpr int UPD_THREADS = 256;  // two warps per TMEM lane quarter: the epilogue is an HBM stream

__global__ void __launch_bounds__(UPD_THREADS) upd_kernel(const __grid_constant__ CUtensorMap ta,
                                                          const __grid_constant__ CUtensorMap tb, StepArgs a,
                                                          UpdArgs p, const StepRow* rows) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Ring R;
  uint8_t* smem = smem_base(smem_raw);
  const StepRow sr = rows[blockIdx.z];
  const int i0 = blockIdx.x * TM, u0 = blockIdx.y * UN;
  const int nu = min(UN, p.fout - u0);
  const int nmma = rup(nu, 16), nbox = (nu + 63) / 64;
  const int kchunks = max(1, (sr.rows + KC - 1) / KC);
  const uint32_t stage_bytes = A_BYTES + (uint32_t)nbox * 8192u;
  if (threadIdx.x == 0) {
    tma::prefetch_map(&ta);
    tma::prefetch_map(&tb);
  }
  ring_init(R, 256);
  if (threadIdx.x == 0) {
    for (int kc = 0; kc < kchunks; ++kc) {
      const int s = kc % 2;
      const uint32_t ph = (uint32_t)(kc / 2) & 1u;
      if (kc >= 2) tc::mbar_wait(&R.empty[s], ph ^ 1u);
      uint8_t* A = smem + s * (A_BYTES + 4 * 8192);
      uint8_t* B = A + A_BYTES;
      tma::expect_tx(&R.full[s], stage_bytes);
      tma::load_3d(A, &ta, i0, kc * KC, sr.slot, &R.full[s]);
      tma::load_3d(A + 8192, &ta, i0 + 64, kc * KC, sr.slot, &R.full[s]);
      for (int j = 0; j < nbox; ++j) tma::load_3d(B + j * 8192, &tb, u0 + 64 * j, kc * KC, sr.slot, &R.full[s]);
    }
  } else if ((threadIdx.x >> 5) == 1) {  // warp 1 issues, converged (mma_bf16_ws: elect.sync)
    const uint32_t idesc = tc::idesc_bf16(TM, nmma, true, true);
    for (int kc = 0; kc < kchunks; ++kc) {
      const int s = kc % 2;
      const uint32_t ph = (uint32_t)(kc / 2) & 1u;
      tc::mbar_wait(&R.full[s], ph);
      tc::fence_after_sync();
      const uint32_t A = tc::smem_u32(smem + s * (A_BYTES + 4 * 8192)), B = A + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < KC / 16; ++kk)
        tc::mma_bf16_ws(R.tmem, tma::mnmajor(A, kk, 8192u), tma::mnmajor(B, kk, 8192u), idesc, (kc | kk) != 0);
      tc::mma_commit_ws(&R.empty[s]);
    }
    tc::mma_commit_ws(&R.done);
  }
  __syncwarp();
  tc::mbar_wait(&R.done, 0);
  tc::fence_after_sync();

  // W_l[i][u] -= lr * G[i][u] on the fp32 master and its bf16 copy. Warp w
  // owns TMEM lane quarter w & 3 (32 rows i) and every other 32-column chunk
  // starting at w >> 2. Each chunk goes TMEM -> registers (lane = row) ->
  // shared memory (the free operand ring) -> registers as 4 rows x 8 float4
  // per instruction, so every global access of a warp covers whole 128-byte
  // row segments; the next chunk's master loads are issued before the
  // current chunk's stores.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = warp & 3;
  const int nchunk = (nmma + 31) / 32;
  const float nlr = -sr.lr;
  float* T = reinterpret_cast<float*>(smem) + warp * (32 * 36);  // [32 rows][36] staging, 144-byte rows
  const int rr0 = lane >> 3, cc = (lane & 7) * 4;                 // pass p: row 4p + rr0, columns cc..cc+3
  float* wbase = a.w_out + (int64_t)sr.req * a.ldw + p.woff + (int64_t)(i0 + q * 32) * p.fout + u0;
  __nv_bfloat16* bbase =
      reinterpret_cast<__nv_bfloat16*>(slot_of(a, sr.slot) + p.wb_off) + (int64_t)(i0 + q * 32) * p.ldw + u0;
  const bool vec = !a.adam && (p.fout % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.w_out + p.woff) & 15) == 0) &&
                   ((a.ldw & 3) == 0) && (p.ldw % 4 == 0);
  auto row_ok = [&](int pp) { return i0 + q * 32 + 4 * pp + rr0 < p.fin; };
  auto col_ok = [&](int c) { return 32 * c + cc + 4 <= nu; };
  float4 cur[8], nxt[8];
  auto load8 = [&](int c, float4 (&d)[8]) {
#pragma unroll
    for (int pp = 0; pp < 8; ++pp)
      if (row_ok(pp) && col_ok(c))
        d[pp] = *reinterpret_cast<const float4*>(wbase + (int64_t)(4 * pp + rr0) * p.fout + 32 * c + cc);
  };
  int c = warp >> 2;
  if (vec && c < nchunk) load8(c, cur);
  for (; c < nchunk; c += 2) {
    const bool has_next = vec && c + 2 < nchunk;
    if (has_next) load8(c + 2, nxt);
    float g[32];
    tc::tmem_ld32(lane_addr(R.tmem, 32 * c), g);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      *reinterpret_cast<float4*>(T + lane * 36 + 4 * k) = make_float4(g[4 * k], g[4 * k + 1], g[4 * k + 2], g[4 * k + 3]);
    __syncwarp();
    if (a.adam) {  // opt-in Adam: moments read-modify-written beside the master (scalar path)
#pragma unroll 1
      for (int pp = 0; pp < 8; ++pp) {
        if (!row_ok(pp)) continue;
        const int row = 4 * pp + rr0;
        for (int e = 0; e < 4; ++e) {
          const int u = 32 * c + cc + e;
          if (u >= nu) break;
          const int64_t idx = p.woff + (int64_t)(i0 + q * 32 + row) * p.fout + u0 + u;
          float* wp = wbase + (int64_t)row * p.fout + u;
          const float w = opt_apply(a, sr, idx, *wp, T[row * 36 + cc + e]);
          *wp = w;
          bbase[(int64_t)row * p.ldw + u] = __float2bfloat16_rn(w);
        }
      }
    } else if (vec) {
#pragma unroll
      for (int pp = 0; pp < 8; ++pp) {
        if (!row_ok(pp)) continue;
        const int row = 4 * pp + rr0;
        if (col_ok(c)) {
          const float4 g4 = *reinterpret_cast<const float4*>(T + row * 36 + cc);
          float4 w = cur[pp];
          w.x = fmaf(nlr, g4.x, w.x);
          w.y = fmaf(nlr, g4.y, w.y);
          w.z = fmaf(nlr, g4.z, w.z);
          w.w = fmaf(nlr, g4.w, w.w);
          *reinterpret_cast<float4*>(wbase + (int64_t)row * p.fout + 32 * c + cc) = w;
          *reinterpret_cast<uint2*>(bbase + (int64_t)row * p.ldw + 32 * c + cc) =
              make_uint2(tc::pack_bf16x2(w.x, w.y), tc::pack_bf16x2(w.z, w.w));
        } else {
          for (int e = 0; e < 4; ++e) {
            const int u = 32 * c + cc + e;
            if (u >= nu) break;
            float* wp = wbase + (int64_t)row * p.fout + u;
            const float w = fmaf(nlr, T[row * 36 + cc + e], *wp);
            *wp = w;
            bbase[(int64_t)row * p.ldw + u] = __float2bfloat16_rn(w);
          }
        }
      }
    } else {
#pragma unroll 1
      for (int pp = 0; pp < 8; ++pp) {
        if (!row_ok(pp)) continue;
        const int row = 4 * pp + rr0;
        for (int e = 0; e < 4; ++e) {
          const int u = 32 * c + cc + e;
          if (u >= nu) break;
          float* wp = wbase + (int64_t)row * p.fout + u;
          const float w = fmaf(nlr, T[row * 36 + cc + e], *wp);
          *wp = w;
          bbase[(int64_t)row * p.ldw + u] = __float2bfloat16_rn(w);
        }
      }
    }
    __syncwarp();
    if (has_next) {
#pragma unroll
      for (int pp = 0; pp < 8; ++pp) cur[pp] = nxt[pp];
    }
  }
  ring_free(R, 256);
}

inline int fwd_smem(int nb) { return 1024 + STAGES * (int)(A_BYTES + nb * 128); }
inline int upd_smem() { return 1024 + 2 * (int)(A_BYTES + 4 * 8192); }
inline int mat_smem() { return 1024 + 2 * (int)(A_BYTES + (UNF / 64) * 8192); }

}  // namespace wide

namespace wide {
// factored-mode history bound of a descriptor (0: dense only): SGD, a known
// max_rows, and epochs x max_rows history rows well under the widest layer
static int fact_bound(const fs_train_desc* d, const MlpLayout& L) {
  if (d->optimizer != FS_OPT_SGD || d->max_rows < 1 || d->epochs < 1) return 0;
  const int64_t h = (int64_t)d->epochs * d->max_rows;
  int wmax = 0;
  for (int l = 1; l < L.L; ++l) wmax = std::max(wmax, L.f[l]);
  return (h <= FACT_MAX_HIST && 2 * h <= wmax) ? (int)h : 0;
}
static size_t stage_bytes(size_t G) { return 256 + G * sizeof(StepRow) + 4 * G + 64 * FACT_VERSIONS + 1024; }
}  // namespace wide

size_t wide_workspace_bytes(const fs_train_desc* d) {
  wide::Geo g;
  if (!d || d->n_req < 1 || !wide::make(d, &g)) return 0;
  const size_t G = (size_t)std::min(d->n_req, wide::WIDE_GROUP);
  size_t need = G * g.slot_bytes + wide::stage_bytes(G);
  if (const int h = wide::fact_bound(d, g.lay)) {
    wide::Geo gf;
    wide::make(d, &gf, h);
    const size_t Gf = (size_t)std::min(d->n_req, wide::FACT_GROUP);
    need = std::max(need, Gf * gf.slot_bytes + wide::FACT_VERSIONS * gf.ver_bytes + wide::stage_bytes(Gf));
  }
  return need;
}

namespace wide {
// the factored lockstep trainer (see the header comment); the caller checked
// SGD, one lr per client, <= FACT_VERSIONS start models and the history bound
static int train_factored(const fs_train_desc* d, const Geo& g, StepArgs sa, const std::vector<int32_t>& nr,
                          const std::vector<int32_t>& bt, const std::vector<int32_t>& s0,
                          const std::vector<int32_t>& s1, const std::vector<double>& lr,
                          const std::vector<uint64_t>& wst, cudaStream_t st) {
  const MlpLayout& L = g.lay;
  const int n = d->n_req, H = g.H, EL = std::max(d->epochs, 1);
  const size_t G = (size_t)std::min(n, FACT_GROUP);
  uint8_t* ws = reinterpret_cast<uint8_t*>(d->workspace);
  uint8_t* slots = ws;
  uint8_t* vers = ws + G * g.slot_bytes;
  uint8_t* stage = vers + FACT_VERSIONS * g.ver_bytes;
  sa.slots = slots;
  sa.g = g;
  // distinct start models -> version blocks (bf16 W0 shared by their clients)
  std::vector<uint64_t> vsrc;
  std::vector<int> vslot(n);
  for (int r = 0; r < n; ++r) {
    auto it = std::find(vsrc.begin(), vsrc.end(), wst[r]);
    vslot[r] = (int)(it - vsrc.begin());
    if (it == vsrc.end()) vsrc.push_back(wst[r]);
  }
  const int nver = (int)vsrc.size();
  {
    cudaMemcpyAsync(stage, vsrc.data(), 8 * (size_t)nver, cudaMemcpyHostToDevice, st);
    VerArgs va;
    va.lay = L;
    va.H = H;
    for (int l = 0; l < MAXL; ++l) {
      va.ldw[l] = g.ldw[l];
      va.wb_off[l] = g.wb_off[l];
    }
    va.ver_bytes = g.ver_bytes;
    va.vers = vers;
    va.src = reinterpret_cast<const uint64_t*>(stage);
    version_convert_kernel<<<dim3(256, (unsigned)nver), 256, 0, st>>>(va);
    if (int rc = check_launch("wide version convert")) return rc;
  }
  ensure_smem(fwd_kernel, fwd_smem(g.nb));
  ensure_smem(bwd_kernel, fwd_smem(g.nb));
  ensure_smem(gram_kernel, fwd_smem(g.nb));
  ensure_smem(mat_kernel, mat_smem());
  int64_t hid_base[MAXL + 1] = {0};
  for (int l = 2; l <= H; ++l) hid_base[l] = hid_base[l - 1] + L.f[l - 1];
  // tensor maps over the version blocks (start weights)
  CUtensorMap fA[MAXL], bA[MAXL];
  bool ok = true;
  for (int l = 0; l < H; ++l) {
    const void* wb = vers + g.wb_off[l];
    ok = ok && tma::make_map(&fA[l], wb, L.f[l + 1], L.f[l], nver, g.ldw[l], g.ver_bytes, 64);
    if (l >= 1) ok = ok && tma::make_map(&bA[l], wb, L.f[l + 1], L.f[l], nver, g.ldw[l], g.ver_bytes, 128);
  }
  uint8_t* stage2 = stage + 64 * FACT_VERSIONS;  // StepRow[] and request ids
  for (int g0 = 0; g0 < n; g0 += (int)G) {
    const int gn = std::min((int)G, n - g0);
    // per-slot maps: history rows (B of the main term, A of the history term
    // and of the grams), P/Q
    CUtensorMap hB[MAXL + 1], hA128[MAXL + 1], hA64[MAXL + 1], dB[MAXL + 1], dA128[MAXL + 1], dA64[MAXL + 1], pq;
    for (int l = 0; l <= H && ok; ++l) {
      const int w = L.f[l];
      const void* hl = slots + g.h_off[l];
      ok = ok && tma::make_map(&hB[l], hl, w, g.rha, gn, g.ld[l], g.slot_bytes, g.nb);
      ok = ok && tma::make_map(&hA128[l], hl, w, g.rha, gn, g.ld[l], g.slot_bytes, 128);
      ok = ok && tma::make_map(&hA64[l], hl, w, g.rha, gn, g.ld[l], g.slot_bytes, 64);
      if (l >= 1) {
        const void* dl = slots + g.d_off[l];
        ok = ok && tma::make_map(&dB[l], dl, w, g.rha, gn, g.ld[l], g.slot_bytes, g.nb);
        ok = ok && tma::make_map(&dA128[l], dl, w, g.rha, gn, g.ld[l], g.slot_bytes, 128);
        ok = ok && tma::make_map(&dA64[l], dl, w, g.rha, gn, g.ld[l], g.slot_bytes, 64);
      }
    }
    ok = ok && tma::make_map(&pq, slots + g.pq_off, g.ldpq, g.rb, gn, g.ldpq, g.slot_bytes, g.nb);
    if (!ok) {
      set_error("fs_train_bf16 (wide, factored): tensor map encoding failed");
      return FS_ECUDA;
    }
    // every history row may be read before this launch writes it (the last
    // K chunk of a history term): zero the group's slots once
    if (cudaMemsetAsync(slots, 0, (size_t)gn * g.slot_bytes, st) != cudaSuccess) return check_launch("wide zero");
    {
      std::vector<int> reqs(gn);
      for (int i = 0; i < gn; ++i) reqs[i] = g0 + i;
      cudaMemcpyAsync(stage2, reqs.data(), 4 * (size_t)gn, cudaMemcpyHostToDevice, st);
      init_small_kernel<<<dim3(4, (unsigned)gn), 256, 0, st>>>(d->w_start, reinterpret_cast<const int*>(stage2), gn,
                                                             L, sa.w_out, d->ldw);
      if (int rc = check_launch("wide init")) return rc;
    }
    std::vector<int> off(gn, 0);
    int t_end = 0, t_begin = INT32_MAX;
    for (int i = 0; i < gn; ++i) {
      t_end = std::max(t_end, s1[g0 + i]);
      t_begin = std::min(t_begin, s0[g0 + i]);
    }
    std::vector<StepRow> rows;
    for (int t = t_begin; t < t_end; ++t) {
      rows.clear();
      int max_off = 0;
      for (int i = 0; i < gn; ++i) {
        const int r = g0 + i;
        if (t < s0[r] || t >= s1[r]) continue;
        const int spe = (nr[r] + bt[r] - 1) / bt[r];
        StepRow sr{};
        sr.req = r;
        sr.slot = i;
        sr.e = t / spe;
        sr.s = t % spe;
        sr.rows = std::min(bt[r], nr[r] - sr.s * bt[r]);
        sr.global_step = t;
        sr.lr = (float)lr[(size_t)r * EL + sr.e];
        sr.off = off[i];
        sr.wslot = vslot[r];
        max_off = std::max(max_off, sr.off);
        off[i] += sr.rows;
        rows.push_back(sr);
      }
      const int A = (int)rows.size();
      if (A == 0) continue;
      cudaMemcpyAsync(stage2, rows.data(), sizeof(StepRow) * A, cudaMemcpyHostToDevice, st);
      const StepRow* d_rows = reinterpret_cast<const StepRow*>(stage2);
      gather_kernel<<<A, 256, 0, st>>>(sa, d_rows);
      if (int rc = check_launch("wide gather")) return rc;
      const unsigned qt = (unsigned)((max_off + TM - 1) / TM);
      // ---- forward
      for (int l = 0; l < H; ++l) {
        if (qt) {
          const GramArgs gp{(L.f[l] + KC - 1) / KC, g.nb, g.pq_off, g.ldpq};
          gram_kernel<<<dim3(qt, (unsigned)g.rtiles, (unsigned)A), THREADS, fwd_smem(g.nb), st>>>(
              hA128[l], hB[l], sa, gp, d_rows);
          if (int rc = check_launch("wide gram")) return rc;
        }
        FwdArgs f{};
        f.l = l + 1;
        f.fin = L.f[l];
        f.fout = L.f[l + 1];
        f.nb = g.nb;
        f.kchunks = (f.fin + KC - 1) / KC;
        f.last = l + 1 == H;
        f.zp = zparts(L.f[H]);
        f.boff = L.boff[l];
        f.whoff = L.woff[H];
        f.hid_base = hid_base[l + 1];
        f.h_off = g.h_off[l + 1];
        f.z_off = g.z_off;
        f.ld_out = g.ld[l + 1];
        fwd_kernel<<<dim3((unsigned)((f.fout + TM - 1) / TM), (unsigned)g.rtiles, (unsigned)A), THREADS,
                     fwd_smem(g.nb), st>>>(fA[l], hB[l], dA64[l + 1], pq, sa, f, d_rows);
        if (int rc = check_launch("wide fwd")) return rc;
      }
      head_kernel<<<A, 256, (size_t)g.rb * 4, st>>>(sa, d_rows);
      if (int rc = check_launch("wide head")) return rc;
      // ---- backward (no per-step weight update: the history is the update)
      for (int l = H - 1; l >= 1; --l) {
        if (qt) {
          const GramArgs gp{(L.f[l + 1] + KC - 1) / KC, g.nb, g.pq_off, g.ldpq};
          gram_kernel<<<dim3(qt, (unsigned)g.rtiles, (unsigned)A), THREADS, fwd_smem(g.nb), st>>>(
              dA128[l + 1], dB[l + 1], sa, gp, d_rows);
          if (int rc = check_launch("wide gram")) return rc;
        }
        BwdArgs p{};
        p.l = l;
        p.fin = L.f[l];
        p.fout = L.f[l + 1];
        p.nb = g.nb;
        p.kchunks = (p.fout + KC - 1) / KC;
        p.boff = L.boff[l - 1];
        p.h_off = g.h_off[l];
        p.d_off = g.d_off[l];
        p.bp_off = g.bp_off[l];
        p.ld = g.ld[l];
        bwd_kernel<<<dim3((unsigned)((p.fin + TM - 1) / TM), (unsigned)g.rtiles, (unsigned)A), THREADS,
                     fwd_smem(g.nb), st>>>(bA[l], dB[l + 1], hA64[l], pq, sa, p, d_rows);
        if (int rc = check_launch("wide bwd")) return rc;
        if (g.rtiles > 1) {
          bias_reduce_kernel<<<dim3((unsigned)((p.fin + 255) / 256), (unsigned)A), 256, 0, st>>>(sa, d_rows, p.fin,
                                                                                                p.boff, p.bp_off);
          if (int rc = check_launch("wide bias")) return rc;
        }
      }
    }
    // ---- the trained rows: W = W0 - lr Hhist^T Dhist, once per client
    rows.clear();
    for (int i = 0; i < gn; ++i) {
      StepRow sr{};
      const int r = g0 + i;
      sr.req = r;
      sr.slot = i;
      sr.off = off[i];
      const int e0 = s0[r] < s1[r] ? s0[r] / ((nr[r] + bt[r] - 1) / bt[r]) : 0;
      sr.lr = (float)lr[(size_t)r * EL + std::min(e0, EL - 1)];
      rows.push_back(sr);
    }
    cudaMemcpyAsync(stage2, rows.data(), sizeof(StepRow) * gn, cudaMemcpyHostToDevice, st);
    const StepRow* d_rows = reinterpret_cast<const StepRow*>(stage2);
    for (int l = 0; l < H; ++l) {
      const MatArgs m{L.f[l], L.f[l + 1], L.woff[l]};
      mat_kernel<<<dim3((unsigned)((m.fin + TM - 1) / TM), (unsigned)((m.fout + UNF - 1) / UNF), (unsigned)gn),
                   UPD_THREADS_F, mat_smem(), st>>>(hA64[l], dA64[l + 1], sa, m, d_rows);
      if (int rc = check_launch("wide mat")) return rc;
    }
  }
  return FS_OK;
}
}  // namespace wide

int wide_train(const fs_train_desc* d, const void* features_bf16, const float* labels, cudaStream_t st) {
  using namespace wide;
  Geo g;
  if (!make(d, &g)) {
    set_error("fs_train_bf16 (wide): invalid layer dims");
    return FS_EINVAL;
  }
  const MlpLayout& L = g.lay;
  const int n = d->n_req;
  if (n == 0) return FS_OK;
  const size_t need = wide_workspace_bytes(d);
  if (!d->workspace || d->workspace_bytes < need) {
    set_error("fs_train_bf16 (wide): workspace %zu < required %zu", d->workspace_bytes, need);
    return FS_EINVAL;
  }
  // per-request geometry on the host (the descriptor's arrays live in HBM)
  std::vector<int32_t> nr(n), bt(n), s0(n), s1(n);
  std::vector<double> lr((size_t)n * std::max(d->epochs, 1));
  cudaMemcpyAsync(nr.data(), d->n_rows, 4 * (size_t)n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(bt.data(), d->batch, 4 * (size_t)n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(s0.data(), d->start_step, 4 * (size_t)n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(s1.data(), d->end_step, 4 * (size_t)n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(lr.data(), d->lr, 8 * lr.size(), cudaMemcpyDeviceToHost, st);
  std::vector<uint64_t> wst(n, 0);
  if (d->w_start) cudaMemcpyAsync(wst.data(), d->w_start, 8 * (size_t)n, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("wide: metadata");
  for (int r = 0; r < n; ++r)
    if (bt[r] > g.rb || bt[r] < 1) {
      set_error("fs_train_bf16 (wide): batch %d exceeds max_batch", bt[r]);
      return FS_EINVAL;
    }

  const size_t G = (size_t)std::min(n, WIDE_GROUP);
  uint8_t* ws = reinterpret_cast<uint8_t*>(d->workspace);
  uint8_t* slots = ws;
  uint8_t* stage = ws + G * g.slot_bytes;  // device staging: StepRow[] (+ request ids at setup)
  float* w_out = reinterpret_cast<float*>(d->w_out);
  const int H = g.H;

  StepArgs sa;
  sa.lay = L;
  sa.g = g;
  sa.slots = slots;
  sa.w_out = w_out;
  sa.ldw = d->ldw;
  sa.feat = reinterpret_cast<const __nv_bfloat16*>(features_bf16);
  sa.labels = labels;
  sa.row_off = d->row_off;
  sa.n_rows = d->n_rows;
  sa.batch = d->batch;
  sa.perm = d->perm;
  sa.perm_off = d->perm_off;
  sa.mask_bits = d->mask_bits;
  sa.mask_off = d->mask_off;
  sa.mask_mode = d->mask_mode;
  sa.scale = (float)d->scale;
  sa.status = d->status;
  sa.adam = d->optimizer == FS_OPT_ADAM;
  sa.b1 = (float)d->adam_beta1;
  sa.b2 = (float)d->adam_beta2;
  sa.eps = (float)d->adam_eps;
  sa.opt = reinterpret_cast<float*>(d->opt_state);
  if (sa.adam && (!sa.opt || d->adam_eps <= 0.0)) {
    set_error("fs_train_bf16 (wide): Adam needs opt_state and eps > 0");
    return FS_EINVAL;
  }
  sa.w_start = d->w_start;
  // factored mode when the launch qualifies (one lr per client, few start
  // models, histories within the workspace's bound); else dense lockstep
  if (const int bound = fact_bound(d, L)) {
    const int EL = std::max(d->epochs, 1);
    bool fact = d->w_start != nullptr;
    int hmax = 0;
    std::vector<uint64_t> seen;
    for (int r = 0; r < n && fact; ++r) {
      const int spe = (nr[r] + bt[r] - 1) / bt[r];
      int h = 0;
      for (int t = s0[r]; t < s1[r]; ++t) {
        h += std::min(bt[r], nr[r] - (t % spe) * bt[r]);
        if (lr[(size_t)r * EL + t / spe] != lr[(size_t)r * EL + s0[r] / spe]) fact = false;
      }
      hmax = std::max(hmax, h);
      if (std::find(seen.begin(), seen.end(), wst[r]) == seen.end()) seen.push_back(wst[r]);
    }
    fact = fact && hmax <= bound && (int)seen.size() <= FACT_VERSIONS;
    if (fact) {
      Geo gf;
      make(d, &gf, bound);
      return train_factored(d, gf, sa, nr, bt, s0, s1, lr, wst, st);
    }
  }
  ConvArgs ca;
  ca.lay = L;
  ca.H = H;
  for (int l = 0; l < MAXL; ++l) {
    ca.ldw[l] = g.ldw[l];
    ca.wb_off[l] = g.wb_off[l];
  }
  ca.slot_bytes = g.slot_bytes;
  ca.slots = slots;
  ca.w_out = w_out;
  ca.ldw_out = d->ldw;

  ensure_smem(fwd_kernel, fwd_smem(g.nb));
  ensure_smem(bwd_kernel, fwd_smem(g.nb));
  ensure_smem(upd_kernel, upd_smem());
  int64_t hid_base[MAXL + 1] = {0};
  for (int l = 2; l <= H; ++l) hid_base[l] = hid_base[l - 1] + L.f[l - 1];

  for (int g0 = 0; g0 < n; g0 += (int)G) {
    const int gn = std::min((int)G, n - g0);
    // tensor maps over this group's slots (slot addresses are fixed for the group)
    CUtensorMap fA[MAXL], fB[MAXL], bA[MAXL], bB[MAXL], uA[MAXL], uB[MAXL];
    bool ok = true;
    for (int l = 0; l < H; ++l) {
      const int fin = L.f[l], fout = L.f[l + 1];
      const void* wb = slots + g.wb_off[l];
      const void* hl = slots + g.h_off[l];
      const void* dn = slots + g.d_off[l + 1];
      ok = ok && tma::make_map(&fA[l], wb, fout, fin, gn, g.ldw[l], g.slot_bytes, 64);
      ok = ok && tma::make_map(&fB[l], hl, fin, g.rb, gn, g.ld[l], g.slot_bytes, g.nb);
      ok = ok && tma::make_map(&uA[l], hl, fin, g.rb, gn, g.ld[l], g.slot_bytes, 64);
      ok = ok && tma::make_map(&uB[l], dn, fout, g.rb, gn, g.ld[l + 1], g.slot_bytes, 64);
      if (l >= 1) {
        ok = ok && tma::make_map(&bA[l], wb, fout, fin, gn, g.ldw[l], g.slot_bytes, 128);
        ok = ok && tma::make_map(&bB[l], dn, fout, g.rb, gn, g.ld[l + 1], g.slot_bytes, g.nb);
      }
    }
    if (!ok) {
      set_error("fs_train_bf16 (wide): tensor map encoding failed");
      return FS_ECUDA;
    }
    // masters <- start rows, then bf16 copies of every slot
    {
      std::vector<StepRow> all(gn);
      for (int i = 0; i < gn; ++i) {
        all[i] = StepRow{};
        all[i].req = g0 + i;
        all[i].slot = i;
      }
      std::vector<int> reqs(gn);
      for (int i = 0; i < gn; ++i) reqs[i] = g0 + i;
      const size_t rbytes = (sizeof(StepRow) * gn + 255) / 256 * 256;
      std::vector<uint8_t> host(rbytes + 4 * (size_t)gn);
      memcpy(host.data(), all.data(), sizeof(StepRow) * gn);
      memcpy(host.data() + rbytes, reqs.data(), 4 * (size_t)gn);
      cudaMemcpyAsync(stage, host.data(), host.size(), cudaMemcpyHostToDevice, st);
      dim3 grid((unsigned)std::min<int64_t>((L.M + 255) / 256, 64), (unsigned)gn);
      init_master_kernel<<<grid, 256, 0, st>>>(d->w_start, reinterpret_cast<const int*>(stage + rbytes), gn, L.M,
                                               w_out, d->ldw);
      if (int rc = check_launch("wide init")) return rc;
      if (sa.adam &&  // moments of this group's requests start at zero
          cudaMemsetAsync(sa.opt + (int64_t)g0 * 2 * d->ldw, 0, sizeof(float) * (size_t)gn * 2 * d->ldw, st) !=
              cudaSuccess)
        return check_launch("wide adam moments");
      convert_kernel<<<dim3(128, (unsigned)gn), 256, 0, st>>>(ca, reinterpret_cast<const StepRow*>(stage), gn);
      if (int rc = check_launch("wide convert")) return rc;
    }
    int t_end = 0;
    for (int i = 0; i < gn; ++i) t_end = std::max(t_end, s1[g0 + i]);
    int t_begin = t_end;
    for (int i = 0; i < gn; ++i) t_begin = std::min(t_begin, s0[g0 + i]);
    for (int t = t_begin; t < t_end; ++t) {
      std::vector<StepRow> rows;
      for (int i = 0; i < gn; ++i) {
        const int r = g0 + i;
        if (t < s0[r] || t >= s1[r]) continue;
        const int spe = (nr[r] + bt[r] - 1) / bt[r];
        StepRow sr{};
        sr.req = r;
        sr.slot = i;
        sr.e = t / spe;
        sr.s = t % spe;
        sr.rows = std::min(bt[r], nr[r] - sr.s * bt[r]);
        sr.global_step = t;
        sr.lr = (float)lr[(size_t)r * std::max(d->epochs, 1) + sr.e];
        rows.push_back(sr);
      }
      const int A = (int)rows.size();
      if (A == 0) continue;
      cudaMemcpyAsync(stage, rows.data(), sizeof(StepRow) * A, cudaMemcpyHostToDevice, st);
      const StepRow* d_rows = reinterpret_cast<const StepRow*>(stage);
      gather_kernel<<<A, 256, 0, st>>>(sa, d_rows);
      if (int rc = check_launch("wide gather")) return rc;
      // ---- forward
      for (int l = 0; l < H; ++l) {
        FwdArgs f{};
        f.l = l + 1;
        f.fin = L.f[l];
        f.fout = L.f[l + 1];
        f.nb = g.nb;
        f.kchunks = (f.fin + KC - 1) / KC;
        f.last = l + 1 == H;
        f.zp = zparts(L.f[H]);
        f.boff = L.boff[l];
        f.whoff = L.woff[H];
        f.hid_base = hid_base[l + 1];
        f.h_off = g.h_off[l + 1];
        f.z_off = g.z_off;
        f.ld_out = g.ld[l + 1];
        fwd_kernel<<<dim3((unsigned)((f.fout + TM - 1) / TM), (unsigned)g.rtiles, (unsigned)A), THREADS,
                     fwd_smem(g.nb), st>>>(fA[l], fB[l], fA[l], fB[l], sa, f, d_rows);
        if (int rc = check_launch("wide fwd")) return rc;
      }
      head_kernel<<<A, 256, (size_t)g.rb * 4, st>>>(sa, d_rows);
      if (int rc = check_launch("wide head")) return rc;
      // ---- backward through W_l (old bf16 copy), then that layer's update
      for (int l = H - 1; l >= 0; --l) {
        if (l >= 1) {
          BwdArgs p{};
          p.l = l;
          p.fin = L.f[l];
          p.fout = L.f[l + 1];
          p.nb = g.nb;
          p.kchunks = (p.fout + KC - 1) / KC;
          p.boff = L.boff[l - 1];
          p.h_off = g.h_off[l];
          p.d_off = g.d_off[l];
          p.bp_off = g.bp_off[l];
          p.ld = g.ld[l];
          bwd_kernel<<<dim3((unsigned)((p.fin + TM - 1) / TM), (unsigned)g.rtiles, (unsigned)A), THREADS,
                       fwd_smem(g.nb), st>>>(bA[l], bB[l], bA[l], bB[l], sa, p, d_rows);
          if (int rc = check_launch("wide bwd")) return rc;
          if (g.rtiles > 1) {
            bias_reduce_kernel<<<dim3((unsigned)((p.fin + 255) / 256), (unsigned)A), 256, 0, st>>>(
                sa, d_rows, p.fin, p.boff, p.bp_off);
            if (int rc = check_launch("wide bias")) return rc;
          }
        }
        UpdArgs u{};
        u.l = l;
        u.fin = L.f[l];
        u.fout = L.f[l + 1];
        u.woff = L.woff[l];
        u.wb_off = g.wb_off[l];
        u.ldw = g.ldw[l];
        upd_kernel<<<dim3((unsigned)((u.fin + TM - 1) / TM), (unsigned)((u.fout + UN - 1) / UN), (unsigned)A),
                     UPD_THREADS, upd_smem(), st>>>(uA[l], uB[l], sa, u, d_rows);
        if (int rc = check_launch("wide upd")) return rc;
      }
    }
  }
  return FS_OK;
}


// ------------------------------------------------------------------ eval forward (wide layers)
namespace wide {

// bf16 copy of W_l [fin x fout] with row stride ldw
__global__ void to_bf16_kernel(const float* src, int fin, int fout, int ldw, __nv_bfloat16* dst) {
  const int64_t total = (int64_t)fin * fout;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = j / fout, u = j - i * fout;
    dst[i * ldw + u] = __float2bfloat16_rn(src[j]);
  }
}

__global__ void eval_probs_kernel(const float* z, int zp, const float* bh, int rows, double* probs) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  float zs = 0.f;
  for (int k = 0; k < zp; ++k) zs += z[(int64_t)r * zp + k];
  const float zz = zs + bh[0];
  probs[r] = (double)(zz >= 0.f ? 1.f / (1.f + __expf(-zz)) : __expf(zz) / (1.f + __expf(zz)));
}

constexpr int EVAL_NB = 128;

struct EvalGeo {
  int dp, ldmax, ldw[MAXL];
  size_t wb_off[MAXL], wb_bytes, act_bytes, z_bytes;
};

static EvalGeo eval_geo(const MlpLayout& L, int rows) {
  EvalGeo e{};
  e.dp = rup(L.f[0], 16);
  size_t o = 0;
  for (int l = 0; l < L.L - 1; ++l) {
    e.ldw[l] = rup(L.f[l + 1], 8);
    e.wb_off[l] = o;
    o += ((size_t)L.f[l] * e.ldw[l] * 2 + 255) / 256 * 256;
  }
  e.wb_bytes = o;
  e.ldmax = rup(std::max(L.max_hidden, 8), 8);
  e.act_bytes = ((size_t)rows * e.ldmax * 2 + 255) / 256 * 256;
  e.z_bytes = (size_t)rows * zparts(L.f[L.L - 1]) * 4 + 256;
  return e;
}

}  // namespace wide
}  // namespace fs

using namespace fs;

extern "C" size_t fs_forward_wide_workspace_bytes(const int32_t* dims, int32_t n_dims, int32_t rows) {
  MlpLayout L;
  if (make_layout(dims, n_dims, &L) != FS_OK || rows < 0 || L.L < 2) return 0;
  const wide::EvalGeo e = wide::eval_geo(L, rows);
  return e.wb_bytes + 2 * e.act_bytes + e.z_bytes;
}

// K8 forward for layer shapes beyond the on-chip kernels (bf16 operands,
// fp32 accumulation, fp32 head): probs_out[rows] of fs_prep_features_bf16
// rows, through the same tcgen05 forward kernel as the wide trainer.
extern "C" int fs_forward_wide(const int32_t* dims, int32_t n_dims, const float* w, const void* x_bf16, int32_t rows,
                               double* probs_out, void* workspace, size_t workspace_bytes, void* stream) {
  using namespace wide;
  MlpLayout L;
  if (make_layout(dims, n_dims, &L) != FS_OK || rows < 0 || L.L < 2) {
    set_error("fs_forward_wide: invalid dims or rows");
    return FS_EINVAL;
  }
  if (rows == 0) return FS_OK;
  const size_t need = fs_forward_wide_workspace_bytes(dims, n_dims, rows);
  if (!workspace || workspace_bytes < need) {
    set_error("fs_forward_wide: workspace %zu < required %zu", workspace_bytes, need);
    return FS_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const EvalGeo e = eval_geo(L, rows);
  uint8_t* p = reinterpret_cast<uint8_t*>(workspace);
  __nv_bfloat16* hbuf[2] = {reinterpret_cast<__nv_bfloat16*>(p + e.wb_bytes),
                            reinterpret_cast<__nv_bfloat16*>(p + e.wb_bytes + e.act_bytes)};
  float* z = reinterpret_cast<float*>(p + e.wb_bytes + 2 * e.act_bytes);
  const int H = L.L - 1;
  ensure_smem(fwd_kernel, fwd_smem(EVAL_NB));
  StepArgs sa{};
  sa.lay = L;
  sa.mask_mode = FS_MASK_NONE;
  const void* in = x_bf16;
  int ld_in = e.dp;
  for (int l = 0; l < H; ++l) {
    const int fin = L.f[l], fout = L.f[l + 1];
    __nv_bfloat16* wl = reinterpret_cast<__nv_bfloat16*>(p + e.wb_off[l]);
    to_bf16_kernel<<<256, 256, 0, st>>>(w + L.woff[l], fin, fout, e.ldw[l], wl);
    if (int rc = check_launch("fs_forward_wide convert")) return rc;
    CUtensorMap ta, tb;
    if (!tma::make_map(&ta, wl, fout, fin, 1, e.ldw[l], 0, 64) ||
        !tma::make_map(&tb, in, fin, rows, 1, ld_in, 0, EVAL_NB)) {
      set_error("fs_forward_wide: tensor map encoding failed");
      return FS_ECUDA;
    }
    const int ld_out = rup(fout, 8);
    FwdArgs f{};
    f.l = l + 1;
    f.fin = fin;
    f.fout = fout;
    f.nb = EVAL_NB;
    f.kchunks = (fin + KC - 1) / KC;
    f.last = l + 1 == H;
    f.zp = zparts(L.f[H]);
    f.boff = L.boff[l];
    f.whoff = L.woff[H];
    f.ld_out = ld_out;
    f.eval = 1;
    f.rows_eval = rows;
    f.h_eval = hbuf[l & 1];
    f.z_eval = z;
    f.w_eval = w;
    fwd_kernel<<<dim3((unsigned)((fout + TM - 1) / TM), (unsigned)((rows + EVAL_NB - 1) / EVAL_NB), 1), THREADS,
                 fwd_smem(EVAL_NB), st>>>(ta, tb, ta, tb, sa, f, nullptr);
    if (int rc = check_launch("fs_forward_wide layer")) return rc;
    in = hbuf[l & 1];
    ld_in = ld_out;
  }
  eval_probs_kernel<<<(rows + 255) / 256, 256, 0, st>>>(z, zparts(L.f[H]), w + L.boff[H], rows, probs_out);
  return check_launch("fs_forward_wide probs");
}
