// K5 (bf16 mixed-precision mode): batched per-client local SGD on the
// 5th-generation tensor cores.
//
// Same contract as the fp64 trainer (client.train_local, client.py:98-172;
// loss_and_grad, _core.pyx:140-219) with mixed precision: fp32 master
// weights (the client's update row, updated in place), bf16 GEMM operands,
// fp32 accumulation in TMEM, fp32 head/loss/SGD arithmetic.
//
// One persistent CTA per SM owns one client at a time (longest first).
// Per SGD step the batch is processed in chunks of 64 rows; every layer
// product is a tcgen05.mma (M=128, N<=256, K=16 slices) issued by one thread
// with operands in shared memory and the accumulator in TMEM:
//   forward   H_{l+1} = relu(H_l W_l + b_l) * mask     (A K-major, B MN-major)
//   backward  G_l     = H_l^T D_{l+1}                  (A MN-major, B MN-major)
//             D_l     = gate(D_{l+1} W_l^T, H_l)       (A K-major, B K-major)
// All bf16 matrices live in shared memory as 8x8 core-matrix tiles, which
// serve both K-major and MN-major operand roles (fs_tc.cuh), so no
// transposes are ever materialised. Epilogues read TMEM with tcgen05.ld,
// apply bias/relu/dropout or the gate, and write bf16 tiles back in place;
// the weight-gradient epilogue applies W -= lr*G to the fp32 master row and
// refreshes the bf16 weight tile. The sigmoid/BCE head (N=1) and the bias
// gradients run on CUDA cores.
#include "fs_bf16.cuh"

namespace fs {
namespace bf16 {

using namespace tc;

struct MaskSrc {
  const uint32_t* bits;  // slot of this step (nullptr = no dropout)
  int step_rows;         // rows of the whole batch (draw layout)
  int row0;              // chunk offset inside the batch
  float scale;
  __device__ __forceinline__ uint32_t word(int64_t j) const { return __ldg(bits + (j >> 5)); }
  // 16 keep bits for (row r of the chunk, units c..c+15) of hidden layer with
  // draw base `base` and width `w`
  __device__ __forceinline__ uint32_t keep16(int base, int r, int c, int w) const {
    const int64_t j = (int64_t)step_rows * base + (int64_t)(row0 + r) * w + c;
    const uint64_t lo = word(j);
    const uint64_t both = ((j >> 5) == ((j + 15) >> 5)) ? lo : (lo | ((uint64_t)word(j + 15) << 32));
    return (uint32_t)(both >> (j & 31)) & 0xFFFFu;
  }
};

// Builds the bf16 tile of weight layer l from the fp32 master row.
__device__ void load_weight_tile(const Geo& g, const float* W, int l, uint8_t* smem) {
  const Tile t{smem_u32(smem + g.s_w[l]), g.fp[l]};
  const int rows = g.fp[l], cols = g.f[l + 1];
  const int chunks = rows * (cols / 8);
  for (int i = threadIdx.x; i < chunks; i += THREADS) {
    const int r = i / (cols / 8), c = (i % (cols / 8)) * 8;
    uint32_t p[4] = {0, 0, 0, 0};
    if (r < g.f[l]) {
      const float* src = W + g.woff[l] + (int64_t)r * cols + c;
#pragma unroll
      for (int k = 0; k < 4; ++k) p[k] = pack_bf16x2(src[2 * k], src[2 * k + 1]);
    }
    st_shared_v4(t.saddr + t.off(r, c), p[0], p[1], p[2], p[3]);
  }
}

// Column sums over the chunk's rows of a bf16 activation tile (bias gradients).
__device__ __forceinline__ float tile_colsum(const Tile& t, int c, int rows) {
  float acc = 0.f;
  const uint32_t colbase = t.saddr + t.off(0, c & ~7) + (uint32_t)((c & 7) * 2);
  for (int r = 0; r < rows; ++r) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(colbase + (uint32_t)((r >> 3) * 128 + (r & 7) * 16)));
    acc += __uint_as_float((uint32_t)v << 16);
  }
  return acc;
}

// Row epilogue of a backward stage: D = gate(acc, H) * dropout * factor,
// written as bf16 in place of H. The accumulator comes from an M=64 MMA, whose
// rows sit 16 per TMEM lane quarter (row q*16 + i at lane 32*q + i), so all 8
// warps work: lanes 0-15 of warp (q, h) own row q*16+lane, column half h.
__device__ __forceinline__ void gate_rows(const Tile& ht, uint32_t tacc, int K, int rows, bool dropout, float scale,
                                          float factor, int q, int h, int lane) {
  const int r = q * 16 + lane;
  const bool own = lane < 16;
  for (int c = h * (K / 2); c < (h + 1) * (K / 2); c += 16) {
    float v[16];
    tmem_ld16(tacc + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
    if (!own) continue;
    uint32_t hv[8];
    ld_shared_v4(ht.saddr + ht.off(r, c), hv[0], hv[1], hv[2], hv[3]);
    ld_shared_v4(ht.saddr + ht.off(r, c + 8), hv[4], hv[5], hv[6], hv[7]);
    const float f = dropout ? factor * scale : factor;
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float lo = bf16lo(hv[k]) > 0.f ? v[2 * k] * f : 0.f;
      float hi = bf16hi(hv[k]) > 0.f ? v[2 * k + 1] * f : 0.f;
      if (r >= rows) lo = hi = 0.f;
      o[k] = pack_bf16x2(lo, hi);
    }
    st_shared_v4(ht.saddr + ht.off(r, c), o[0], o[1], o[2], o[3]);
    st_shared_v4(ht.saddr + ht.off(r, c + 8), o[4], o[5], o[6], o[7]);
  }
}

// Backward through the 3 hidden layers with on-chip optimizer state (V2).
// Layer indices: W_0 [f0 x f1] (HBM master), W_1 [f1 x f2] (TMEM master),
// W_2 [f2 x f3] (smem master). D_3 (unscaled) is in the H_3 slot on entry.
__device__ __forceinline__ void backward_v2(const Geo& g, const Args& a, uint8_t* smem, uint32_t tbase, uint32_t& phase,
                                         uint64_t& mma_bar, float* W, float* bias_sh, float lr, int rows,
                                         bool last_chunk, bool dropout, float scale, int tid, int q, int h,
                                         int lane, unsigned long long* s_prof, long long& prof_t0) {
  const int f0 = g.f[0], fp0 = g.fp[0], f1 = g.f[1], f2 = g.f[2], f3 = g.f[3];
  const int mb1 = (f1 + 127) / 128;
  const Tile xt{smem_u32(smem + g.s_h[0]), R};
  const Tile h1{smem_u32(smem + g.s_h[1]), R};
  const Tile h2{smem_u32(smem + g.s_h[2]), R};
  const Tile h3{smem_u32(smem + g.s_h[3]), R};
  const Tile w0t{smem_u32(smem + g.s_w[0]), fp0};
  const Tile w1t{smem_u32(smem + g.s_w[1]), f1};
  const Tile w2t{smem_u32(smem + g.s_w[2]), f2};
  float* w2m = reinterpret_cast<float*>(smem + g.s_w2m);

  // ---------------- stage 2: G2 = H2^T D3 (TMEM [0,f3)), D2 = D3 W2^T (TMEM [f3, f3+f2))
  stage_sync();
  if (tid == 0) {
    const uint32_t idg = idesc_bf16(128, f3, true, true);
    for (int ks = 0; ks < R / 16; ++ks) mma_bf16(tbase, h2.mnmajor(ks), h3.mnmajor(ks), idg, ks > 0);
    const uint32_t idd = idesc_bf16(64, f2, false, false);
    for (int ks = 0; ks < f3 / 16; ++ks) mma_bf16(tbase + (uint32_t)f3, h3.kmajor(ks), w2t.kmajor(ks), idd, ks > 0);
    mma_commit(&mma_bar);
  }
  wait_mma(&mma_bar, phase);
  FS_PROF(14);
  // D2 carries the step size from here on: tiles hold -lr * dL/dH
  gate_rows(h2, tbase + (uint32_t)f3, f2, rows, dropout, scale, -lr, q, h, lane);
  FS_PROF(18);
  {  // W2 -= lr * G2 on the shared-memory master (column-major: lane-consecutive rows)
    const int m = q * 32 + lane;
    for (int c = h * (f3 / 2); c < (h + 1) * (f3 / 2); c += 16) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
      if (m < f2) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float* p = w2m + (c + i) * f2 + m;
          const float nw = *p - lr * v[i];
          *p = nw;
          v[i] = nw;
        }
        if (last_chunk) {
          st_shared_v4(w2t.saddr + w2t.off(m, c), pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                       pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
          st_shared_v4(w2t.saddr + w2t.off(m, c + 8), pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]),
                       pack_bf16x2(v[12], v[13]), pack_bf16x2(v[14], v[15]));
        }
      }
    }
  }
  for (int c = tid; c < f3; c += THREADS) {  // b2 -= lr * colsum(D3)
    const float nb = W[g.boff[2] + c] - lr * tile_colsum(h3, c, rows);
    W[g.boff[2] + c] = nb;
    if (last_chunk) bias_sh[g.bias_off[2] + c] = nb;
  }
  FS_PROF(22);

  // ---------------- stage 1: W1_master += H1^T (-lr D2) in TMEM; D1 = (-lr D2) W1^T (TMEM [0,f1))
  stage_sync();
  if (tid == 0) {
    const uint32_t idg = idesc_bf16(128, f2, true, true);
    for (int mb = 0; mb < mb1; ++mb)
      for (int ks = 0; ks < R / 16; ++ks)
        mma_bf16(tbase + 256u + (uint32_t)(mb * f2), h1.mnmajor(ks, mb), h2.mnmajor(ks), idg, 1u);
    const uint32_t idd = idesc_bf16(64, f1, false, false);
    for (int ks = 0; ks < f2 / 16; ++ks) mma_bf16(tbase, h2.kmajor(ks), w1t.kmajor(ks), idd, ks > 0);
    mma_commit(&mma_bar);
  }
  wait_mma(&mma_bar, phase);
  FS_PROF(13);
  gate_rows(h1, tbase, f1, rows, dropout, scale, 1.f, q, h, lane);
  FS_PROF(17);
  if (last_chunk) {  // refresh the bf16 W1 tile from the TMEM master
    for (int mb = 0; mb < mb1; ++mb) {
      const int m = mb * 128 + q * 32 + lane;
      for (int c = h * (f2 / 2); c < (h + 1) * (f2 / 2); c += 16) {
        float v[16];
        tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + 256u + (uint32_t)(mb * f2 + c), v);
        if (m < f1) {
          st_shared_v4(w1t.saddr + w1t.off(m, c), pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                       pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
          st_shared_v4(w1t.saddr + w1t.off(m, c + 8), pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]),
                       pack_bf16x2(v[12], v[13]), pack_bf16x2(v[14], v[15]));
        }
      }
    }
  }
  for (int c = tid; c < f2; c += THREADS) {  // b1 += colsum(-lr D2)
    const float nb = W[g.boff[1] + c] + tile_colsum(h2, c, rows);
    W[g.boff[1] + c] = nb;
    if (last_chunk) bias_sh[g.bias_off[1] + c] = nb;
  }
  FS_PROF(21);

  // ---------------- stage 0: G0^T = (-lr D1)^T X (TMEM [mb*fp0, ...)), W0 += G0^T^T in HBM
  stage_sync();
  if (tid == 0) {
    const uint32_t idg = idesc_bf16(128, fp0, true, true);
    for (int mb = 0; mb < mb1; ++mb)
      for (int ks = 0; ks < R / 16; ++ks)
        mma_bf16(tbase + (uint32_t)(mb * fp0), h1.mnmajor(ks, mb), xt.mnmajor(ks), idg, ks > 0);
    mma_commit(&mma_bar);
  }
  // W0 master slices (coalesced across lanes) for both M-blocks, issued before
  // the TMEM reads so their latency overlaps the gradient MMA drain
  constexpr int MAXCI = 2;  // 16-column chunks per thread and M-block (fp0 <= 64)
  float wpre[2][MAXCI][16];
#pragma unroll
  for (int mb = 0; mb < 2; ++mb) {
    const int m = mb * 128 + q * 32 + lane;
#pragma unroll
    for (int j = 0; j < MAXCI; ++j) {
      const int c = (h + 2 * j) * 16;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        wpre[mb][j][i] = (mb < mb1 && m < f1 && c + i < f0) ? W[(c + i) * f1 + m] : 0.f;
    }
  }
  wait_mma(&mma_bar, phase);
  FS_PROF(12);
#pragma unroll
  for (int mb = 0; mb < 2; ++mb) {
    if (mb >= mb1) break;
    const int m = mb * 128 + q * 32 + lane;  // output unit of layer 0
#pragma unroll
    for (int j = 0; j < MAXCI; ++j) {
      const int c = (h + 2 * j) * 16;
      if (c >= fp0) break;
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(mb * fp0 + c), v);
      if (m < f1) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (c + i < f0) {
            const float w = wpre[mb][j][i] + v[i];
            W[(c + i) * f1 + m] = w;
            if (last_chunk) {
              const __nv_bfloat16 b = __float2bfloat16_rn(w);
              const uint32_t ad = w0t.saddr + w0t.off(c + i, m & ~7) + (uint32_t)((m & 7) * 2);
              asm volatile("st.shared.b16 [%0], %1;" ::"r"(ad), "h"(*reinterpret_cast<const uint16_t*>(&b)));
            }
          }
        }
      }
    }
  }
  for (int c = tid; c < f1; c += THREADS) {  // b0 += colsum(-lr D1)
    const float nb = W[g.boff[0] + c] + tile_colsum(h1, c, rows);
    W[g.boff[0] + c] = nb;
    if (last_chunk) bias_sh[g.bias_off[0] + c] = nb;
  }
  FS_PROF(20);
}

// V2 = on-chip optimizer state for 3-hidden-layer MLPs: the largest hidden
// weight's fp32 master lives in TMEM columns [256, 512) and is updated by the
// weight-gradient MMA itself (master += H^T (-lr D)); W_{L-2}'s master lives
// in shared memory; W_0's master stays in HBM but is updated through the
// transposed gradient G_0^T so every warp issues coalesced row segments.
template <bool V2>
__global__ void __maxnreg__(FS_BF16_MAXNREG) train_bf16_kernel(Args a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mma_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_item;
  __shared__ int64_t s_rowidx[R];
  __shared__ int64_t s_rowidx_next[R];
  __shared__ float s_y_next[R];
  __shared__ unsigned long long s_prof[32];
  long long prof_t0 = clock64();

  const Geo& g = a.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, h = warp >> 2;
  float* misc = reinterpret_cast<float*>(smem + g.s_misc);
  float* z_sh = misc;              // [R]
  float* dz_sh = misc + R;         // [R]
  float* y_sh = misc + 2 * R;      // [R]
  float* zpart = misc + 3 * R;     // [2][R]
  float* gwh = misc + 5 * R;       // [f_{L-1}] head weight grad (<= 256)
  float* gbh = misc + 5 * R + 256; // [1]
  float* bias_sh = reinterpret_cast<float*>(smem + g.s_bias);

  if (tid < 32) s_prof[tid] = 0;
  if (warp == 0) tmem_alloc(&tmem_base_sh, TMEM_COLS);
  if (tid == 0) {
    mbar_init(&mma_bar, 1);
    fence_mbar_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = tmem_base_sh;
  uint32_t phase = 0;
  float* gacc = a.gacc + (int64_t)blockIdx.x * g.M;
  const int L = g.L;
  const int FL = g.f[L - 1];  // width feeding the head

  while (true) {
    if (tid == 0) s_item = atomicAdd(a.counter, 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= a.n_req) break;
    const int rq = a.order[item];
    const int n = a.n_rows[rq], B = a.batch[rq];
    const int spe = (n + B - 1) / B;
    float* W = a.w_out + (int64_t)rq * a.ldw;
    const float* W0 = reinterpret_cast<const float*>(a.w_start[rq]);
    if (W0 != W) {  // 16-byte vector copy of the start parameters (rows are 16 B aligned)
      const int nv = g.M / 4;
      const float4* s4 = reinterpret_cast<const float4*>(W0);
      float4* d4 = reinterpret_cast<float4*>(W);
      if ((reinterpret_cast<uintptr_t>(W0) & 15) == 0) {
        for (int j = tid; j < nv; j += 4 * THREADS) {
          float4 t[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j + u * THREADS < nv) t[u] = __ldg(s4 + j + u * THREADS);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j + u * THREADS < nv) d4[j + u * THREADS] = t[u];
        }
        for (int j = 4 * nv + tid; j < g.M; j += THREADS) W[j] = W0[j];
      } else {
        for (int j = tid; j < g.M; j += THREADS) W[j] = W0[j];
      }
    }
    __syncthreads();
    for (int l = 0; l < L - 1; ++l) {
      load_weight_tile(g, W, l, smem);
      for (int j = tid; j < g.f[l + 1]; j += THREADS) bias_sh[g.bias_off[l] + j] = W[g.boff[l] + j];
    }
    if constexpr (V2) {
      // W_1 master -> TMEM [256, 512); W_2 master -> smem (column-major)
      const int f1 = g.f[1], f2 = g.f[2], f3 = g.f[3];
      for (int mb = 0; mb < (g.fp[1] + 127) / 128; ++mb) {
        const int m = mb * 128 + q * 32 + lane;
        for (int c = h * (f2 / 2); c < (h + 1) * (f2 / 2); c += 16) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = m < f1 ? W[g.woff[1] + m * f2 + c + i] : 0.f;
          tmem_st16(tbase + ((uint32_t)(q * 32) << 16) + 256u + (uint32_t)(mb * f2 + c), v);
        }
      }
      float* w2m = reinterpret_cast<float*>(smem + g.s_w2m);
      for (int i = tid; i < f2 * f3; i += THREADS) w2m[(i % f3) * f2 + i / f3] = W[g.woff[2] + i];
    }
    // padding columns of the input tile stay zero forever (gather writes only f0)
    const int64_t slot_words = ((int64_t)B * g.sum_hidden + 31) / 32;
    bool have_next = false;
    uint4 xnext[XPRE];

    for (int step = a.start_step[rq]; step < a.end_step[rq]; ++step) {
      const int e = step / spe, s = step % spe;
      const int step_rows = min(B, n - s * B);
      const float lr = (float)a.lr[(int64_t)rq * a.epochs + e];
      const int32_t* perm_e = a.perm + a.perm_off[rq] + (int64_t)e * n;
      MaskSrc mk;
      mk.bits = a.mask_mode == FS_MASK_BITS ? a.mask_bits + a.mask_off[rq] + (int64_t)step * slot_words : nullptr;
      mk.step_rows = step_rows;
      mk.scale = a.scale;
      const int nchunks = (step_rows + R - 1) / R;

      for (int ch = 0; ch < nchunks; ++ch) {
        const int row0 = ch * R;
        const int rows = min(R, step_rows - row0);
        const bool last_chunk = ch == nchunks - 1;
        const bool first_chunk = ch == 0;
        mk.row0 = row0;
        // ---------------- gather the chunk's rows (bf16 features) and labels;
        // after the first chunk of a client they were prefetched during the
        // previous chunk's backward pass (registers xnext / smem *_next)
        const int cpr = g.fp[0] / 8;  // 16-byte chunks per input row
        if (have_next) {
          if (tid < R) {
            s_rowidx[tid] = s_rowidx_next[tid];
            y_sh[tid] = s_y_next[tid];
          }
        } else if (tid < R) {
          const int64_t row = tid < rows ? a.row_off[rq] + perm_e[s * B + row0 + tid] : -1;
          s_rowidx[tid] = row;
          y_sh[tid] = row >= 0 ? a.labels[row] : 0.f;
        }
        __syncthreads();
        FS_PROF(0);
        {
          const Tile xt{smem_u32(smem + g.s_h[0]), R};
#pragma unroll
          for (int u = 0; u < XPRE; ++u) {
            const int i = tid + u * THREADS;
            if (i < R * cpr) {
              const int r = i / cpr, c = (i % cpr) * 8;
              uint4 v = xnext[u];
              if (!have_next) {
                v = make_uint4(0, 0, 0, 0);
                if (r < rows) v = __ldg(reinterpret_cast<const uint4*>(a.feat + s_rowidx[r] * g.fp[0] + c));
              }
              st_shared_v4(xt.saddr + xt.off(r, c), v.x, v.y, v.z, v.w);
            }
          }
        }
        have_next = false;
        // next chunk of this client (same step or the next one)
        int nstep = step, nch = ch + 1;
        if (nch == nchunks) {
          nstep = step + 1;
          nch = 0;
        }
        const bool next_ok = nstep < a.end_step[rq];
        // ---------------- forward through the hidden layers
        int base = 0;  // mask draw base of hidden layer l
        for (int l = 0; l < L - 1; ++l) {
          const int K = g.fp[l], N = g.f[l + 1];
          stage_sync();
          if (tid == 0) {
            const Tile at{smem_u32(smem + g.s_h[l]), R};
            const Tile bt{smem_u32(smem + g.s_w[l]), g.fp[l]};
            const uint32_t id = idesc_bf16(64, N, false, true);
            for (int ks = 0; ks < K / 16; ++ks) mma_bf16(tbase, at.kmajor(ks), bt.mnmajor(ks), id, ks > 0);
            mma_commit(&mma_bar);
          }
          // keep-bits of this thread's (row, column half) fetched while the MMA runs
          uint32_t mw[5] = {0, 0, 0, 0, 0};
          int mbit0 = 0;
          if (mk.bits && lane < 16) {
            const int64_t j0 = (int64_t)mk.step_rows * base + (int64_t)(row0 + q * 16 + lane) * N + h * (N / 2);
            const int64_t w0 = j0 >> 5, w1 = (j0 + N / 2 - 1) >> 5;
            mbit0 = (int)(j0 & 31);
#pragma unroll
            for (int i = 0; i < 5; ++i)
              if (w0 + i <= w1) mw[i] = __ldg(mk.bits + w0 + i);
          }
          wait_mma(&mma_bar, phase);
          FS_PROF(1 + l);
          // epilogue (M=64 accumulator layout): lanes 0-15 of warp (q, h) own
          // row q*16+lane, columns [h*N/2, (h+1)*N/2); all 8 warps work
          const bool head_in = (l == L - 2);
          float zp = 0.f;
          {
            const int r = q * 16 + lane;
            const bool own = lane < 16;
            const Tile ot{smem_u32(smem + g.s_h[l + 1]), R};
            const float* bias = bias_sh + g.bias_off[l];
            const float* wh = W + g.woff[L - 1];
            for (int c = h * (N / 2); c < (h + 1) * (N / 2); c += 16) {
              float v[16];
              tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
              if (!own) continue;
              uint32_t keep = 0xFFFFu;
              if (mk.bits) {
                const int p = mbit0 + (c - h * (N / 2));
                const int wi = p >> 5, sh = p & 31;
                uint32_t lo = 0, hi = 0;
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                  if (i == wi) lo = mw[i];
                  if (i == wi + 1) hi = mw[i];
                }
                keep = (uint32_t)((((uint64_t)hi << 32) | lo) >> sh) & 0xFFFFu;
              }
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                float x = v[i] + bias[c + i];
                x = x > 0.f ? x : 0.f;
                if (mk.bits) x = ((keep >> i) & 1u) ? x * mk.scale : 0.f;
                if (r >= rows) x = 0.f;
                v[i] = x;
              }
              if (head_in) {
#pragma unroll
                for (int i = 0; i < 16; ++i) zp = fmaf(v[i], __ldg(wh + c + i), zp);
              }
              st_shared_v4(ot.saddr + ot.off(r, c), pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                           pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
              st_shared_v4(ot.saddr + ot.off(r, c + 8), pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]),
                           pack_bf16x2(v[12], v[13]), pack_bf16x2(v[14], v[15]));
            }
            if (head_in && own) zpart[h * R + r] = zp;
          }
          FS_PROF(5 + l);
          base += N;
        }
        if (next_ok && tid < R) {  // prefetch A: next chunk's row ids and labels
          const int ne = nstep / spe, ns = nstep % spe;
          const int nrows_step = min(B, n - ns * B);
          const int nr0 = nch * R;
          const int64_t row = tid < min(R, nrows_step - nr0)
                                  ? a.row_off[rq] + a.perm[a.perm_off[rq] + (int64_t)ne * n + ns * B + nr0 + tid]
                                  : -1;
          s_rowidx_next[tid] = row;
          s_y_next[tid] = row >= 0 ? a.labels[row] : 0.f;
        }
        // ---------------- head: logits, dz = (sigmoid(z) - y) / step_rows
        stage_sync();
        if (tid < R) {
          const float z = zpart[tid] + zpart[R + tid] + W[g.boff[L - 1]];
          z_sh[tid] = z;
          float d = 0.f;
          if (tid < rows) {
            d = (sigmoidf_stable(z) - y_sh[tid]) / (float)step_rows;
            if (!isfinite(z)) atomicOr(a.status + rq, 1);
          }
          dz_sh[tid] = d;
        }
        __syncthreads();
        FS_PROF(9);
        if (next_ok) {  // prefetch B: next chunk's feature rows, held in registers
#pragma unroll
          for (int u = 0; u < XPRE; ++u) {
            const int i = tid + u * THREADS;
            xnext[u] = make_uint4(0, 0, 0, 0);
            if (i < R * cpr) {
              const int64_t row = s_rowidx_next[i / cpr];
              if (row >= 0) xnext[u] = __ldg(reinterpret_cast<const uint4*>(a.feat + row * g.fp[0] + (i % cpr) * 8));
            }
          }
          have_next = true;
        }
        // head weight/bias gradients (from the bf16 H_{L-1} tile, fp32 sums)
        {
          const Tile ht{smem_u32(smem + g.s_h[L - 1]), R};
          for (int k = tid; k < FL; k += THREADS) {
            float acc = 0.f;
            const uint32_t colbase = ht.saddr + ht.off(0, k & ~7) + (uint32_t)((k & 7) * 2);
            for (int r = 0; r < rows; ++r) {
              uint16_t hv;
              asm volatile("ld.shared.u16 %0, [%1];" : "=h"(hv) : "r"(colbase + (uint32_t)((r >> 3) * 128 + (r & 7) * 16)));
              acc = fmaf(__uint_as_float((uint32_t)hv << 16), dz_sh[r], acc);
            }
            gwh[k] = acc;
          }
          if (tid == THREADS - 1) {
            float sacc = 0.f;
            for (int r = 0; r < rows; ++r) sacc += dz_sh[r];
            gbh[0] = sacc;
          }
        }
        __syncthreads();
        FS_PROF(10);
        // D_{L-1} = gate(dz (x) w_head, H_{L-1}) written in place of H_{L-1}
        {
          const Tile ht{smem_u32(smem + g.s_h[L - 1]), R};
          const float* wh = W + g.woff[L - 1];
          const int cpr = FL / 8;
          for (int i = tid; i < R * cpr; i += THREADS) {
            const int r = i / cpr, c = (i % cpr) * 8;
            const uint32_t ad = ht.saddr + ht.off(r, c);
            uint32_t p[4];
            ld_shared_v4(ad, p[0], p[1], p[2], p[3]);
            const float dzr = dz_sh[r];
            uint32_t o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              float lo = bf16lo(p[k]) > 0.f ? dzr * __ldg(wh + c + 2 * k) : 0.f;
              float hi = bf16hi(p[k]) > 0.f ? dzr * __ldg(wh + c + 2 * k + 1) : 0.f;
              if (mk.bits) {
                lo *= mk.scale;
                hi *= mk.scale;
              }
              o[k] = pack_bf16x2(lo, hi);
            }
            st_shared_v4(ad, o[0], o[1], o[2], o[3]);
          }
        }
        // head update (or accumulation for a multi-chunk step), after D used old w
        __syncthreads();
        FS_PROF(11);
        if constexpr (V2) {
          float* wh = W + g.woff[L - 1];
          float* ghs = misc + 5 * R + 260;  // [FL] head-gradient accumulator across chunks
          for (int k = tid; k < FL; k += THREADS) {
            const float gk = gwh[k] + (first_chunk ? 0.f : ghs[k]);
            if (last_chunk) wh[k] = wh[k] - lr * gk; else ghs[k] = gk;
          }
          if (tid == THREADS - 1) {
            const float gb = gbh[0] + (first_chunk ? 0.f : ghs[FL]);
            if (last_chunk) W[g.boff[L - 1]] = W[g.boff[L - 1]] - lr * gb; else ghs[FL] = gb;
          }
        } else {
          float* wh = W + g.woff[L - 1];
          float* ga = gacc + g.woff[L - 1];
          for (int k = tid; k < FL; k += THREADS) {
            const float gk = gwh[k] + (first_chunk ? 0.f : ga[k]);
            if (last_chunk) wh[k] = wh[k] - lr * gk; else ga[k] = gk;
          }
          if (tid == THREADS - 1) {
            const int bo = g.boff[L - 1];
            const float gb = gbh[0] + (first_chunk ? 0.f : gacc[bo]);
            if (last_chunk) W[bo] = W[bo] - lr * gb; else gacc[bo] = gb;
          }
        }
        if constexpr (V2) {
          backward_v2(g, a, smem, tbase, phase, mma_bar, W, bias_sh, lr, rows, last_chunk, mk.bits != nullptr,
                      mk.scale, tid, q, h, lane, s_prof, prof_t0);
        } else
        // ---------------- backward through the hidden layers
        for (int l = L - 2; l >= 0; --l) {
          const int K = g.fp[l];        // rows of W_l (padded)
          const int N = g.f[l + 1];     // cols of W_l
          const int mblocks = (K + 127) / 128;
          const uint32_t dcol = (uint32_t)(mblocks * N);  // TMEM column of D_l
          stage_sync();
          if (tid == 0) {
            const Tile ht{smem_u32(smem + g.s_h[l]), R};       // H_l (X for l = 0)
            const Tile dt{smem_u32(smem + g.s_h[l + 1]), R};   // D_{l+1} (in place of H_{l+1})
            const Tile wt{smem_u32(smem + g.s_w[l]), g.fp[l]};
            const uint32_t idg = idesc_bf16(128, N, true, true);
            for (int mb = 0; mb < mblocks; ++mb)
              for (int ks = 0; ks < R / 16; ++ks)
                mma_bf16(tbase + (uint32_t)(mb * N), ht.mnmajor(ks, mb), dt.mnmajor(ks), idg, ks > 0);
            if (l > 0) {
              const uint32_t idd = idesc_bf16(128, K, false, false);
              for (int ks = 0; ks < N / 16; ++ks) mma_bf16(tbase + dcol, dt.kmajor(ks), wt.kmajor(ks), idd, ks > 0);
            }
            mma_commit(&mma_bar);
          }
          wait_mma(&mma_bar, phase);
          FS_PROF(12 + l);
          // (a) D_l = gate(acc, H_l) in place of H_l  (rows q*32+lane, column half h)
          if (l > 0 && q < 2) {
            const int r = q * 32 + lane;
            const Tile ht{smem_u32(smem + g.s_h[l]), R};
            for (int c = h * (K / 2); c < (h + 1) * (K / 2); c += 16) {
              float v[16];
              tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + dcol + (uint32_t)c, v);
              uint32_t hv[8];
              ld_shared_v4(ht.saddr + ht.off(r, c), hv[0], hv[1], hv[2], hv[3]);
              ld_shared_v4(ht.saddr + ht.off(r, c + 8), hv[4], hv[5], hv[6], hv[7]);
              uint32_t o[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                float lo = bf16lo(hv[k]) > 0.f ? v[2 * k] : 0.f;
                float hi = bf16hi(hv[k]) > 0.f ? v[2 * k + 1] : 0.f;
                if (mk.bits) {
                  lo *= mk.scale;
                  hi *= mk.scale;
                }
                if (r >= rows) lo = hi = 0.f;
                o[k] = pack_bf16x2(lo, hi);
              }
              st_shared_v4(ht.saddr + ht.off(r, c), o[0], o[1], o[2], o[3]);
              st_shared_v4(ht.saddr + ht.off(r, c + 8), o[4], o[5], o[6], o[7]);
            }
          }
          FS_PROF(16 + l);
          // (b) G_l -> W_l -= lr * G_l on the fp32 master row; refresh the bf16 tile
          {
            const Tile wt{smem_u32(smem + g.s_w[l]), g.fp[l]};
            float* Wl = W + g.woff[l];
            float* Gl = gacc + g.woff[l];
            const bool single = first_chunk && last_chunk;
            for (int mb = 0; mb < mblocks; ++mb) {
              const int m = mb * 128 + q * 32 + lane;
              const bool valid = m < g.f[l];
              const int cend = (h + 1) * (N / 2);
              for (int c0 = h * (N / 2); c0 < cend; c0 += 64) {
                const int cw = min(64, cend - c0);  // multiple of 16, warp-uniform
                float4 wv[16];
                if (single && valid) {  // issue the whole master slice before touching TMEM
                  const float4* wp4 = reinterpret_cast<const float4*>(Wl + (int64_t)m * N + c0);
#pragma unroll
                  for (int i = 0; i < 16; ++i)
                    if (4 * i < cw) wv[i] = wp4[i];
                }
#pragma unroll
                for (int s16 = 0; s16 < 4; ++s16) {
                  if (16 * s16 >= cw) break;
                  const int c = c0 + 16 * s16;
                  float v[16];
                  tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(mb * N + c), v);
                  if (!valid) continue;
                  float* wp = Wl + (int64_t)m * N + c;
                  float* gp = Gl + (int64_t)m * N + c;
                  if (!single) {
                    if (!first_chunk) {
#pragma unroll
                      for (int i = 0; i < 16; ++i) v[i] += gp[i];
                    }
                    if (!last_chunk) {
#pragma unroll
                      for (int i = 0; i < 16; ++i) gp[i] = v[i];
                      continue;
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) wv[4 * s16 + i] = reinterpret_cast<const float4*>(wp)[i];
                  }
                  float nw[16];
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    float4 w4 = wv[4 * s16 + i];
                    w4.x -= lr * v[4 * i];
                    w4.y -= lr * v[4 * i + 1];
                    w4.z -= lr * v[4 * i + 2];
                    w4.w -= lr * v[4 * i + 3];
                    reinterpret_cast<float4*>(wp)[i] = w4;
                    nw[4 * i] = w4.x;
                    nw[4 * i + 1] = w4.y;
                    nw[4 * i + 2] = w4.z;
                    nw[4 * i + 3] = w4.w;
                  }
                  st_shared_v4(wt.saddr + wt.off(m, c), pack_bf16x2(nw[0], nw[1]), pack_bf16x2(nw[2], nw[3]),
                               pack_bf16x2(nw[4], nw[5]), pack_bf16x2(nw[6], nw[7]));
                  st_shared_v4(wt.saddr + wt.off(m, c + 8), pack_bf16x2(nw[8], nw[9]),
                               pack_bf16x2(nw[10], nw[11]), pack_bf16x2(nw[12], nw[13]),
                               pack_bf16x2(nw[14], nw[15]));
                }
              }
            }
          }
          FS_PROF(20 + l);
          // (c) bias b_l gradient: column sums of D_{l+1} over the chunk's rows
          {
            const Tile dt{smem_u32(smem + g.s_h[l + 1]), R};
            float* bl = W + g.boff[l];
            float* gb = gacc + g.boff[l];
            for (int c = tid; c < N; c += THREADS) {
              float acc = 0.f;
              const uint32_t colbase = dt.saddr + dt.off(0, c & ~7) + (uint32_t)((c & 7) * 2);
              for (int r = 0; r < rows; ++r) {
                uint16_t dv;
                asm volatile("ld.shared.u16 %0, [%1];" : "=h"(dv) : "r"(colbase + (uint32_t)((r >> 3) * 128 + (r & 7) * 16)));
                acc += __uint_as_float((uint32_t)dv << 16);
              }
              if (!first_chunk) acc += gb[c];
              if (last_chunk) {
                const float nb = bl[c] - lr * acc;
                bl[c] = nb;
                bias_sh[g.bias_off[l] + c] = nb;
              } else {
                gb[c] = acc;
              }
            }
          }
        }
        FS_PROF(24);
        __syncthreads();
        FS_PROF(25);
      }  // chunks
    }    // steps
    if constexpr (V2) {  // write the on-chip masters back to the client's row
      fence_before_sync();
      __syncthreads();
      fence_after_sync();
      const int f1 = g.f[1], f2 = g.f[2], f3 = g.f[3];
      for (int mb = 0; mb < (g.fp[1] + 127) / 128; ++mb) {
        const int m = mb * 128 + q * 32 + lane;
        for (int c = h * (f2 / 2); c < (h + 1) * (f2 / 2); c += 16) {
          float v[16];
          tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + 256u + (uint32_t)(mb * f2 + c), v);
          if (m < f1) {
#pragma unroll
            for (int i = 0; i < 16; i += 4)
              *reinterpret_cast<float4*>(W + g.woff[1] + m * f2 + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          }
        }
      }
      const float* w2m = reinterpret_cast<const float*>(smem + g.s_w2m);
      for (int i = tid; i < f2 * f3; i += THREADS) W[g.woff[2] + i] = w2m[(i % f3) * f2 + i / f3];
      fence_before_sync();
    }
    __syncthreads();
  }
  fence_before_sync();
  __syncthreads();
  if (a.prof && tid < 32) atomicAdd(a.prof + tid, s_prof[tid]);
  if (warp == 0) tmem_dealloc(tbase, TMEM_COLS);
}

// features float64 [rows x d] -> bf16 [rows x dp] zero padded; labels -> fp32
__global__ void prep_features_kernel(const double* X, const double* Y, int64_t rows, int d, int dp,
                                     __nv_bfloat16* xb, float* yf) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * dp) return;
  const int64_t r = i / dp;
  const int c = (int)(i % dp);
  xb[i] = __float2bfloat16_rn(c < d ? (float)X[r * d + c] : 0.f);
  if (c == 0 && yf) yf[r] = (float)Y[r];
}

}  // namespace bf16

using namespace bf16;

int bf16::make_geo(const int32_t* dims, int32_t n_dims, Geo* out) {
  if (n_dims < 3 || n_dims > MAXL + 1) return FS_EINVAL;
  Geo g{};
  g.L = n_dims - 1;
  for (int i = 0; i < n_dims; ++i) g.f[i] = dims[i];
  if (g.f[g.L] != 1 || g.f[0] < 1 || g.f[0] > 64) return FS_EINVAL;  // input rows prefetched in registers
  g.fp[0] = (g.f[0] + 15) / 16 * 16;
  for (int l = 1; l < g.L; ++l) {
    if (g.f[l] % 32 != 0 || g.f[l] < 32 || g.f[l] > 256) return FS_EINVAL;
    g.fp[l] = g.f[l];
  }
  int off = 0;
  for (int l = 0; l < g.L; ++l) {
    g.woff[l] = off;
    off += g.f[l] * g.f[l + 1];
    g.boff[l] = off;
    off += g.f[l + 1];
  }
  g.M = off;
  g.sum_hidden = 0;
  for (int l = 1; l < g.L; ++l) g.sum_hidden += g.f[l];
  if (g.f[g.L - 1] > 256) return FS_EINVAL;
  // TMEM budget of every backward stage: G blocks + D columns
  for (int l = 0; l < g.L - 1; ++l) {
    const int mblocks = (g.fp[l] + 127) / 128;
    const int cols = mblocks * g.f[l + 1] + (l > 0 ? g.fp[l] : 0);
    if (cols > (int)TMEM_COLS) return FS_EINVAL;
  }
  uint32_t s = 0;
  for (int l = 0; l < g.L; ++l) {  // activation tiles (X, H_1..H_{L-1})
    g.s_h[l] = s;
    s += (uint32_t)(R * g.fp[l] * 2);
  }
  for (int l = 0; l < g.L - 1; ++l) {  // hidden weight tiles
    g.s_w[l] = s;
    s += (uint32_t)(g.fp[l] * g.f[l + 1] * 2);
  }
  g.s_misc = s;
  s += (5 * R + 256 + 4 + 260) * 4;  // z, dz, y, zpart[2], gw_head, gb_head, head-grad accumulator
  g.s_bias = s;
  {
    int bo = 0;
    for (int l = 0; l < g.L - 1; ++l) {
      g.bias_off[l] = bo;
      bo += g.f[l + 1];
    }
    s += (uint32_t)((bo + 3) / 4 * 16);
  }
  // V2 (on-chip optimizer state): 3 hidden layers, W_1 master fits TMEM
  // columns [256,512), W_2 master fits shared memory, and every transient
  // accumulator fits TMEM columns [0,256)
  g.v2 = 0;
  if (g.L == 4) {
    const int mb1 = (g.f[1] + 127) / 128;
    const bool tm = mb1 * g.f[2] <= 256 && g.f[1] <= 256 && g.f[2] <= 128 && g.f[3] + g.f[2] <= 256 &&
                    mb1 * g.fp[0] <= 256 && g.fp[0] <= 64 && mb1 <= 2;
    const uint32_t w2m_bytes = (uint32_t)(g.f[2] * g.f[3] * 4);
    if (tm && s + w2m_bytes <= 220 * 1024) {
      g.v2 = 1;
      g.s_w2m = s;
      s += w2m_bytes;
    }
  }
  if (!g.v2) {
    // generic path: MMAs with M=128 over 64-row tiles read up to 16 KB past a
    // tile; keep those reads inside the allocation
    s += 16 * 1024;
  }
  g.smem_bytes = s;
  if (s > 220 * 1024) return FS_EINVAL;
  *out = g;
  return FS_OK;
}

}  // namespace fs

using namespace fs;

static unsigned long long* g_bf16_prof = nullptr;
static int g_bf16_force_generic = 0;

// Diagnostic kernel selection: 0 = automatic (unit-major V3 where the layer
// shape allows, else row-major V2, else generic), 1 = generic (HBM optimizer
// state), 2 = row-major V2.
extern "C" void fs_bf16_force_generic(int mode) { g_bf16_force_generic = mode; }

// Diagnostic: accumulate per-phase SM cycles of the bf16 trainer into a
// device buffer of 32 counters (nullptr disables).
extern "C" void fs_bf16_set_profile(unsigned long long* counters) { g_bf16_prof = counters; }

// 1 = on-chip tensor-core trainers, 2 = wide lockstep trainer (fs_train_wide.cu), 0 = neither
extern "C" int fs_bf16_supported(const int32_t* dims, int32_t n_dims) {
  Geo g;
  if (make_geo(dims, n_dims, &g) == FS_OK) return 1;
  MlpLayout lay;
  if (n_dims >= 3 && n_dims <= FS_MAX_LAYERS + 1 && make_layout(dims, n_dims, &lay) == FS_OK && dims[0] <= 4096)
    return 2;
  return 0;
}

extern "C" int fs_prep_features_bf16(const double* x, const double* y, int64_t rows, int32_t d, int32_t dp,
                                     void* xb_out, float* y_out, void* stream) {
  if (rows < 0 || d < 1 || dp < d || dp % 8) {
    set_error("fs_prep_features_bf16: invalid sizes");
    return FS_EINVAL;
  }
  if (rows == 0) return FS_OK;
  const int64_t total = rows * dp;
  prep_features_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      x, y, rows, d, dp, reinterpret_cast<__nv_bfloat16*>(xb_out), y_out);
  return check_launch("prep_features_kernel");
}

extern "C" int fs_forward_bf16(const int32_t* dims, int32_t n_dims, const float* w, const void* x_bf16,
                               int32_t rows, double* probs_out, void* stream) {
  Geo g;
  if (make_geo(dims, n_dims, &g) != FS_OK || !bf16t::geo_ok(g) || rows < 0) {
    set_error("fs_forward_bf16: unsupported layer dims or rows");
    return FS_EINVAL;
  }
  if (rows == 0) return FS_OK;
  return bf16t::launch_eval(g, w, x_bf16, rows, probs_out, (cudaStream_t)stream);
}

extern "C" size_t fs_train_bf16_workspace_bytes(const fs_train_desc* d) {
  Geo g;
  if (!d || d->n_req < 1) return 0;
  if (d->optimizer == FS_OPT_ADAM)  // the opt-in Adam runs on the wide (lockstep) trainer for every shape
    return fs_bf16_supported(d->dims, d->n_dims) ? wide_workspace_bytes(d) : 0;
  if (make_geo(d->dims, d->n_dims, &g) != FS_OK) return fs_bf16_supported(d->dims, d->n_dims) == 2 ? wide_workspace_bytes(d) : 0;
  const int grid = d->grid > 0 ? d->grid : kNumSMs;
  const int gg = grid < d->n_req ? grid : d->n_req;
  return 256 + (size_t)gg * g.M * sizeof(float);
}

extern "C" int fs_train_bf16(const fs_train_desc* d, const void* features_bf16, const float* labels_f32,
                             void* stream) {
  Geo g;
  if (d && ((make_geo(d->dims, d->n_dims, &g) != FS_OK && fs_bf16_supported(d->dims, d->n_dims) == 2) ||
            (d->optimizer == FS_OPT_ADAM && fs_bf16_supported(d->dims, d->n_dims)))) {
    if (!d->w_start && d->n_req > 0) {
      set_error("fs_train_bf16 (wide): w_start is NULL");
      return FS_EINVAL;
    }
    return wide_train(d, features_bf16, labels_f32, (cudaStream_t)stream);
  }
  if (!d || make_geo(d->dims, d->n_dims, &g) != FS_OK) {
    set_error("fs_train_bf16: unsupported layer dims for the tensor-core trainer");
    return FS_EINVAL;
  }
  if (d->n_req == 0) return FS_OK;
  const size_t need = fs_train_bf16_workspace_bytes(d);
  if (!d->workspace || d->workspace_bytes < need) {
    set_error("fs_train_bf16: workspace %zu < required %zu", d->workspace_bytes, need);
    return FS_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Args a;
  a.g = g;
  a.n_req = d->n_req;
  a.epochs = d->epochs;
  a.mask_mode = d->mask_mode;
  a.scale = (float)d->scale;
  a.feat = reinterpret_cast<const __nv_bfloat16*>(features_bf16);
  a.labels = labels_f32;
  a.row_off = d->row_off;
  a.n_rows = d->n_rows;
  a.batch = d->batch;
  a.lr = d->lr;
  a.w_start = d->w_start;
  a.w_out = reinterpret_cast<float*>(const_cast<double*>(d->w_out));
  a.ldw = d->ldw;
  a.perm = d->perm;
  a.perm_off = d->perm_off;
  a.mask_bits = d->mask_bits;
  a.mask_off = d->mask_off;
  a.start_step = d->start_step;
  a.end_step = d->end_step;
  a.order = d->order;
  a.status = d->status;
  a.counter = reinterpret_cast<int*>(d->workspace);
  a.gacc = reinterpret_cast<float*>(reinterpret_cast<char*>(d->workspace) + 256);
  a.prof = g_bf16_prof;
  a.mask_flags = d->mask_mode == FS_MASK_BITS ? d->mask_flags : nullptr;
  a.mask_tag = d->mask_tag;
  a.max_steps = d->max_steps;
  a.done = d->done;
  a.w_prev = d->w_prev;
  a.counts_out = d->done ? nullptr : d->align_counts;
  a.align_mode = (d->done || d->align_counts) ? d->align_mode : -1;
  a.done_tag = d->done_tag;
  if (a.counts_out && (a.align_mode < 0 || (a.align_mode == FS_ALIGN_DELTA_SIGN && !d->w_prev))) {
    set_error("fs_train_bf16: align_counts needs align_mode (and w_prev for delta_sign)");
    return FS_EINVAL;
  }
  a.data_flags = d->data_flags;
  a.data_chunk = d->data_chunk;
  a.data_tag = d->data_tag;
  if (a.mask_flags) preload_mask_producer();
  if (a.data_flags) preload_flag_publisher();
  a.w_all = reinterpret_cast<const float*>(d->w_start_all);
  const bool v3 = g_bf16_force_generic == 0 && bf16t::geo_ok(g);
  if (!a.w_start && !(v3 && a.w_all)) {
    set_error("fs_train_bf16: w_start is NULL (w_start_all needs the unit-major kernel's layer shapes)");
    return FS_EINVAL;
  }
  if (!(v3 && d->counter_zeroed) && cudaMemsetAsync(a.counter, 0, sizeof(int), st) != cudaSuccess)
    return check_launch("memset");
  int grid = d->grid > 0 ? d->grid : kNumSMs;
  if (grid > d->n_req) grid = d->n_req;
  if (g_bf16_force_generic == 0 && bf16t::geo_ok(g)) return bf16t::launch(a, grid, st);
  if (a.mask_flags || a.done || a.data_flags || a.counts_out) {
    set_error("fs_train_bf16: flagged keep bits / completion records need the unit-major kernel's layer shapes");
    return FS_EINVAL;
  }
  if (g.v2 && g_bf16_force_generic != 1) {
    ensure_smem(train_bf16_kernel<true>, (int)g.smem_bytes);
    train_bf16_kernel<true><<<grid, THREADS, g.smem_bytes, st>>>(a);
  } else {
    if (g.v2) {  // the generic kernel needs its over-read pad
      a.g.smem_bytes += 16 * 1024;
      g.smem_bytes += 16 * 1024;
    }
    ensure_smem(train_bf16_kernel<false>, (int)g.smem_bytes);
    train_bf16_kernel<false><<<grid, THREADS, g.smem_bytes, st>>>(a);
  }
  return check_launch("train_bf16_kernel");
}
