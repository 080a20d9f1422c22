// K5 (bf16 mixed precision), unit-major variant "V3": the product trainer for
// 3-hidden-layer MLPs of the UNSW shape (f1 in {128, 256}, f2 = 128, f3 = 64,
// f0 <= 64). Same contract as fs_train_bf16.cu (client.train_local,
// client.py:98-172 with bf16 GEMM operands and fp32 masters).
//
// Every activation/gradient tile is stored transposed, units x batch rows
// (H^T, D^T), so every tcgen05.mma has M = 128 units and every TMEM
// accumulator row belongs to one unit. An epilogue thread therefore owns one
// unit across 32 batch rows: bias is one register, the bias gradient is a
// per-thread sum, the bf16 tile row it writes is 64 contiguous bytes, and all
// 32 lanes of a warp do useful work (the row-major kernel used half of them).
//
//   forward   H_{l+1}^T = relu(W_l^T H_l^T + b_l) * mask    (M = units, N = 64 rows)
//   head      z = H_3 w_h + b_h   (warp reduce-scatter over units), dz = (sigmoid(z) - y) / rows
//   backward  W_2 -= lr * H_2^T D_3           (G_2 in TMEM -> fp32 master in smem)
//             D_2^T = gate(W_2 D_3^T) * (-lr)
//             W_1 master (TMEM) += H_1^T D_2   (the MMA applies the update)
//             D_1^T = gate(W_1 D_2^T)
//             W_0^T master (TMEM) += D_1^T X   (the MMA applies the update)
//
// Optimizer state never leaves the SM while a client trains: W_0^T and W_1
// masters in TMEM, W_2 / biases / head in shared memory; HBM sees the start
// row once and the trained row once per client.
//
// Dropout keep bits keep K3's (row, unit) draw layout: each lane fetches the
// 32 unit bits of one batch row and a 32x32 warp bit-transpose hands every
// lane the 32 row bits of its unit.
#include "fs_bf16.cuh"

namespace fs {
namespace bf16t {

using namespace tc;
using bf16::Args;
using bf16::Geo;
using bf16::R;
using bf16::THREADS;
using bf16::XPRE;
using bf16::stage_sync;
using bf16::wait_mma;

// TMEM columns (512 allocated)
constexpr uint32_t T_ACC = 0;    // transient accumulators [0, 128)
constexpr uint32_t T_D2 = 64;    // D_2^T accumulator during stage 2 (G_2 uses [0, 64))
constexpr uint32_t T_W0 = 128;   // W_0^T master: M-block mb at [128 + mb*fp0, ...)
constexpr uint32_t T_W1 = 256;   // W_1 master:   M-block mb at [256 + mb*f2, ...)

// fp32 scratch (float offsets inside the `fl` region)
constexpr int FL_Y = 0, FL_DZ = 64, FL_ZP = 128, FL_GW = 256, FL_GB2 = 384, FL_GB1 = 512, FL_GB0 = 768,
              FL_GHS = 1280, FL_GBACC = 1348, FL_BIAS = 1796, FL_WH = 2244, FL_GBH = 2312, FL_N = 2320;

struct Lay {
  uint32_t x, h1, h2, h3, w0, w1, w2, w2m, fl, total;
};

__host__ __device__ inline Lay lay_of(const Geo& g) {
  Lay l;
  uint32_t s = 0;
  l.x = s;   s += (uint32_t)(R * g.fp[0] * 2);
  l.h1 = s;  s += (uint32_t)(g.f[1] * R * 2);
  l.h2 = s;  s += (uint32_t)(g.f[2] * R * 2);
  l.h3 = s;  s += (uint32_t)(g.f[3] * R * 2);
  l.w0 = s;  s += (uint32_t)(g.f[1] * g.fp[0] * 2);
  l.w1 = s;  s += (uint32_t)(g.f[1] * g.f[2] * 2);
  l.w2 = s;  s += (uint32_t)(g.f[2] * g.f[3] * 2);
  // the F2 MMA runs M = 128 over the 64 output units: its A operand reads
  // 16 KB past the W_2 tile, which lands in the (allocated) W_2 master
  l.w2m = s; s += (uint32_t)(g.f[2] * g.f[3] * 4);
  l.fl = s;  s += (uint32_t)(FL_N * 4);
  // (one X tile: a second one, staged during the previous chunk's backward
  // pass, pushes the CTA past the shared memory that lets the next round's
  // K2 blocks co-reside, and the round loses more than the trainer gains)
  l.total = s;
  return l;
}

bool geo_ok(const Geo& g) {
  return g.L == 4 && (g.f[1] == 128 || g.f[1] == 256) && g.f[2] == 128 && g.f[3] == 64 && g.fp[0] <= 64 &&
         lay_of(g).total <= 220 * 1024;
}
uint32_t smem_bytes(const Geo& g) { return lay_of(g).total; }

#define FS_PROF(k)                                        \
  do {                                                    \
    if (a.prof && tid == 0) {                             \
      const long long t1_ = clock64();                    \
      s_prof[k] += (unsigned long long)(t1_ - prof_t0);   \
      prof_t0 = t1_;                                      \
    }                                                     \
  } while (0)

// 32x32 bit-matrix transpose across a warp: in, lane k bit u = A[k][u];
// out, lane u bit k = A[k][u].
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int j = 16; j >= 1; j >>= 1) {
    const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu : j == 2 ? 0x33333333u
                                                                                                     : 0x55555555u;
    const uint32_t t = __shfl_xor_sync(0xFFFFFFFFu, x, j);
    x = (lane & j) ? ((x & ~m) | ((t >> j) & m)) : ((x & m) | ((t << j) & ~m));
  }
  return x;
}

// Warp reduce-scatter: returns sum over lanes of p[lane] (p is clobbered).
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

__device__ __forceinline__ uint32_t rows_valid(int rows, int rb) {
  const int k = rows - rb;
  return k >= 32 ? 0xFFFFFFFFu : (k > 0 ? (1u << k) - 1u : 0u);
}

// Load pinned where it is written (volatile: the compiler may not sink it
// towards its use, which would expose the latency it is meant to hide).
// L2-coherent (.cg): with flagged keep bits the words of a later step may be
// written by the concurrent K3 after an earlier step's read cached the line.
__device__ __forceinline__ uint32_t ldg_early(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Wait until K3 has published the keep bits of (request, step).
__device__ __forceinline__ void wait_mask_step(const int32_t* flag, int32_t tag) {
  if (!flag) return;
  int32_t v;
  uint32_t spins = 0;
  while (true) {
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v == tag) break;
    __nanosleep(128);
    if (++spins > (1u << 24)) __trap();  // a missing producer must not hang the GPU
  }
}

// Raw keep-bit words of this warp's four forward items (F0 block 0, F0
// block 1, F1, F2), issued one chunk ahead so their latency hides behind the
// previous chunk's backward pass.
struct MaskRaw {
  uint32_t lo[4], hi[4];
};

struct ItemGeo {  // item k of warp (q, hh): draw base, layer width, first unit, active
  int base, N, m0, act;
};

__device__ __forceinline__ ItemGeo mask_item(int k, int f1, int f2, int f3, int MB, int q) {
  if (k < 2) return ItemGeo{0, f1, k * 128 + q * 32, k < MB};
  if (k == 2) return ItemGeo{f1, f2, q * 32, 1};
  return ItemGeo{f1 + f2, f3, q * 32, q < f3 / 32};
}

__device__ __forceinline__ void mask_issue(MaskRaw& mr, const uint32_t* bits, int step_rows, int row0, int rows,
                                           int f1, int f2, int f3, int MB, int q, int hh, int lane) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const ItemGeo it = mask_item(k, f1, f2, f3, MB, q);
    mr.lo[k] = mr.hi[k] = 0u;
    if (bits && it.act && hh * 32 + lane < rows) {
      const int64_t j = (int64_t)step_rows * it.base + (int64_t)(row0 + hh * 32 + lane) * it.N + it.m0;
      mr.lo[k] = ldg_early(bits + (j >> 5));
      if (j & 31) mr.hi[k] = ldg_early(bits + (j >> 5) + 1);
    }
  }
}

// keep word of each item: bit r = keep(row hh*32 + r, this lane's unit), rows
// past the chunk cleared
__device__ __forceinline__ void mask_finish(const MaskRaw& mr, bool has_bits, int step_rows, int rows, int f1, int f2,
                                            int f3, int MB, int q, int hh, int lane, uint32_t (&kw)[4]) {
  const uint32_t valid = rows_valid(rows, hh * 32);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const ItemGeo it = mask_item(k, f1, f2, f3, MB, q);
    kw[k] = valid;
    if (has_bits && it.act) {  // warp-uniform
      const int sh = (int)(((int64_t)step_rows * it.base) & 31);  // row*N and m0 are multiples of 32
      const uint32_t x = (uint32_t)((((uint64_t)mr.hi[k] << 32) | mr.lo[k]) >> sh);
      kw[k] &= transpose32(x, lane);
    }
  }
}

__device__ __forceinline__ void store_row32(const Tile& t, int m, int c0, const float (&v)[32]) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    st_shared_v4(t.saddr + t.off(m, c0 + 8 * k), pack_bf16x2(v[8 * k], v[8 * k + 1]),
                 pack_bf16x2(v[8 * k + 2], v[8 * k + 3]), pack_bf16x2(v[8 * k + 4], v[8 * k + 5]),
                 pack_bf16x2(v[8 * k + 6], v[8 * k + 7]));
}

__device__ __forceinline__ void load_row32(const Tile& t, int m, int c0, uint32_t (&hv)[16]) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    ld_shared_v4(t.saddr + t.off(m, c0 + 8 * k), hv[4 * k], hv[4 * k + 1], hv[4 * k + 2], hv[4 * k + 3]);
}

__device__ __forceinline__ float bf16_at(const uint32_t (&hv)[16], int j) {
  return (j & 1) ? bf16hi(hv[j >> 1]) : bf16lo(hv[j >> 1]);
}

// D^T row segment = gate(acc, H^T) * factor written in place of H^T; returns
// the sum of the stored (bf16-rounded) values, i.e. this segment's share of
// the bias gradient.
__device__ __forceinline__ float gate_seg(const Tile& t, int m, int c0, uint32_t taddr, float factor) {
  uint32_t raw[32];
  tmem_ld32_nw(taddr, raw);
  uint32_t hv[16];
  load_row32(t, m, c0, hv);
  tmem_wait_ld_r(raw);
  float d[32];
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float x = bf16_at(hv, j) > 0.f ? __uint_as_float(raw[j]) * factor : 0.f;
    d[j] = x;
  }
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const uint32_t p = pack_bf16x2(d[j], d[j + 1]);
    s += bf16lo(p);
    s += bf16hi(p);
  }
  store_row32(t, m, c0, d);
  return s;
}

__device__ __forceinline__ int sgn_f(float x) { return (x > 0.f) - (x < 0.f); }
__device__ __forceinline__ int sgn_d(float a, float b) { return (a > b) - (a < b); }

// K6 for one freshly trained row (selection.calculate_relevance,
// selection.py:53-74), then {aligned, status, tag} into the client's record
// (system-scope release: the record usually lives in mapped host memory and
// the trained row must be visible to kernels the host launches next).
__device__ __noinline__ void client_done(int M, int mode, const float* W, const float* g, const float* p,
                                         const int32_t* status, uint64_t rec_addr, int32_t tag, int tid,
                                         int64_t* count_out) {
  __shared__ unsigned long long s_cnt[THREADS / 32];
  unsigned cnt = 0;
  if (mode == FS_ALIGN_DELTA_SIGN && !p) mode = -1;  // no movement history: unscored (server.py:283-284)
  if (mode >= 0) {
    // 16-byte loads, four in flight per thread: the row was just written by
    // this CTA (L2), g and p are shared by every client (L2-resident)
    const int M4 = (((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(g) |
                      (p ? reinterpret_cast<uintptr_t>(p) : 0)) & 15) == 0) ? M / 4 : 0;
    const float4* W4 = reinterpret_cast<const float4*>(W);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    const float4* p4 = reinterpret_cast<const float4*>(p);
    if (mode == FS_ALIGN_WEIGHT_SIGN) {
#pragma unroll 4
      for (int j = tid; j < M4; j += THREADS) {
        const float4 c = __ldcg(W4 + j), gv = __ldg(g4 + j);
        cnt += (sgn_f(c.x) == sgn_f(gv.x)) + (sgn_f(c.y) == sgn_f(gv.y)) + (sgn_f(c.z) == sgn_f(gv.z)) +
               (sgn_f(c.w) == sgn_f(gv.w));
      }
    } else {
#pragma unroll 4
      for (int j = tid; j < M4; j += THREADS) {
        const float4 c = __ldcg(W4 + j), gv = __ldg(g4 + j), pv = __ldg(p4 + j);
        cnt += (sgn_d(c.x, gv.x) == sgn_d(gv.x, pv.x)) + (sgn_d(c.y, gv.y) == sgn_d(gv.y, pv.y)) +
               (sgn_d(c.z, gv.z) == sgn_d(gv.z, pv.z)) + (sgn_d(c.w, gv.w) == sgn_d(gv.w, pv.w));
      }
    }
    for (int j = 4 * M4 + tid; j < M; j += THREADS) {
      const float c = __ldcg(W + j), gv = __ldg(g + j);
      cnt += mode == FS_ALIGN_WEIGHT_SIGN ? (sgn_f(c) == sgn_f(gv)) : (sgn_d(c, gv) == sgn_d(gv, __ldg(p + j)));
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((tid & 31) == 0) s_cnt[tid >> 5] = cnt;
  __syncthreads();
  if (tid == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < THREADS / 32; ++w) t += s_cnt[w];
    if (count_out) {  // sync round: a plain count, ordered by the kernel's completion
      *count_out = (int64_t)t;
      return;
    }
    fs_client_done* rec = reinterpret_cast<fs_client_done*>(rec_addr);
    rec->aligned = (int64_t)t;
    rec->status = __ldcg(status);
    __threadfence_system();
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(&rec->tag), "r"(tag) : "memory");
  }
}

// 184 registers x 256 threads leaves room for one 128-thread block of the next
// round's K3 (70 registers) on the same SM. Warp 0 issues every stage's MMAs
// warp-converged (mma_bf16_ws: elect.sync inside the instruction block); a
// single divergent issuing thread (tid == 0) made the compiler serialise each
// tcgen05.mma in a per-lane loop with its descriptors moved to uniform
// registers one by one (~100-240 cycles per MMA; 12.7 -> 12.0 us per 64-row
// step of the C4 world's longest client, scripts/chain_probe.py). A dedicated
// ninth MMA warp was measured too: 3 warps on one SM sub-partition cap the
// registers at 168 and the epilogues then lose more than the issue gains.
#ifndef FS_D3_QUARTERS
#define FS_D3_QUARTERS 1
#endif
#ifndef FS_BF16T_MAXNREG
#define FS_BF16T_MAXNREG 184
#endif
__global__ void __maxnreg__(FS_BF16T_MAXNREG) train_kernel(Args a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mma_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_item;
  // row ids and labels of the current chunk and the prefetched next one,
  // ping-ponged (cur flips when a prefetched chunk becomes current: no copy,
  // no barrier at the chunk start)
  __shared__ int64_t s_rowidx_pp[2][R];
  __shared__ float s_y_pp[2][R];
  __shared__ unsigned long long s_prof[32];
  long long prof_t0 = clock64();

  const Geo& g = a.g;
  const Lay ly = lay_of(g);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = warp & 3;
  const int f0 = g.f[0], fp0 = g.fp[0], f1 = g.f[1], f2 = g.f[2], f3 = g.f[3];
  const int MB = f1 / 128;
  float* fl = reinterpret_cast<float*>(smem + ly.fl);
  float* dz_sh = fl + FL_DZ;
  float* zpart = fl + FL_ZP;    // [2][R]
  float* gwp = fl + FL_GW;      // [2][64] head weight gradient partials
  float* gb2p = fl + FL_GB2;    // [2][64]
  float* gb1p = fl + FL_GB1;    // [2][128]
  float* gb0p = fl + FL_GB0;    // [2][256]
  float* ghs = fl + FL_GHS;     // [f3 + 1] head gradient accumulated over a step's chunks
  float* gbacc = fl + FL_GBACC; // [f1 + f2 + f3] bias gradients accumulated over a step's chunks
  float* bias = fl + FL_BIAS;   // [f1 + f2 + f3] fp32 hidden biases (master and forward copy)
  float* wh = fl + FL_WH;       // [f3 + 1] head weights + bias
  float* gbh = fl + FL_GBH;     // [2] head bias gradient partials
  float* w2m = reinterpret_cast<float*>(smem + ly.w2m);  // W_2 master, column-major [f3][f2]
  const Tile xt{smem_u32(smem + ly.x), R};
  const Tile h1t{smem_u32(smem + ly.h1), f1};
  const Tile h2t{smem_u32(smem + ly.h2), f2};
  const Tile h3t{smem_u32(smem + ly.h3), f3};
  const Tile w0t{smem_u32(smem + ly.w0), f1};  // W_0^T [f1 x fp0]
  const Tile w1t{smem_u32(smem + ly.w1), f1};  // W_1   [f1 x f2]
  const Tile w2t{smem_u32(smem + ly.w2), f2};  // W_2   [f2 x f3]

  if (tid < 32) s_prof[tid] = 0;
  if (warp == 0) tmem_alloc(&tmem_base_sh, bf16::TMEM_COLS);
  if (tid == 0) {
    mbar_init(&mma_bar, 1);
    fence_mbar_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = tmem_base_sh;
  const uint32_t tq = tbase + ((uint32_t)(q * 32) << 16);  // this warp's TMEM lane quarter
  uint32_t phase = 0;

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
    const float* Ws = a.w_start ? reinterpret_cast<const float*>(a.w_start[rq]) : a.w_all;
    if (a.data_flags) wait_mask_step(a.data_flags + a.data_chunk[rq], a.data_tag);  // this client's rows uploaded
    FS_PROF(30);

    // ---------------- client start: masters and bf16 tiles from the start row
    // (every thread issues all of its loads before the first store)
    {
      const int hh = (warp >> 2) & 1;
      // W_1 rows, one M-block per pass: item (mb, q, hh) -> unit m, columns [hh*f2/2, +f2/2);
      // the first pass also carries the W_2 rows (unit q*32+lane, columns [hh*f3/2, +f3/2))
#pragma unroll 1
      for (int k = 0; k < MB; ++k) {
        const int m = k * 128 + q * 32 + lane;
        float4 w1v[16];
        const float4* src = reinterpret_cast<const float4*>(Ws + g.woff[1] + (int64_t)m * f2 + hh * (f2 / 2));
#pragma unroll
        for (int i = 0; i < 16; ++i) w1v[i] = src[i];
        float4 w2v[8];
        if (k == 0) {
          const float4* s2 = reinterpret_cast<const float4*>(Ws + g.woff[2] + (int64_t)(q * 32 + lane) * f3 + hh * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) w2v[i] = s2[i];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c0 = hh * (f2 / 2) + 16 * j;
          float v[16];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            v[4 * i] = w1v[4 * j + i].x; v[4 * i + 1] = w1v[4 * j + i].y;
            v[4 * i + 2] = w1v[4 * j + i].z; v[4 * i + 3] = w1v[4 * j + i].w;
          }
          tmem_st16(tq + T_W1 + (uint32_t)(k * f2 + c0), v);
          st_shared_v4(w1t.saddr + w1t.off(m, c0), pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                       pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
          st_shared_v4(w1t.saddr + w1t.off(m, c0 + 8), pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]),
                       pack_bf16x2(v[12], v[13]), pack_bf16x2(v[14], v[15]));
        }
        if (k == 0) {
          const int m2 = q * 32 + lane;
          float v[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            v[4 * i] = w2v[i].x; v[4 * i + 1] = w2v[i].y; v[4 * i + 2] = w2v[i].z; v[4 * i + 3] = w2v[i].w;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) w2m[(hh * 32 + i) * f2 + m2] = v[i];
          store_row32(w2t, m2, hh * 32, v);
        }
      }
      FS_PROF(31);
      // W_0^T rows: warp w -> block mb = w >> 2, unit m, all fp0 columns (coalesced across lanes)
      const int mb0 = warp >> 2;
      if (mb0 < MB) {
        const int m = mb0 * 128 + q * 32 + lane;
        float w0v[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) w0v[c] = c < f0 ? Ws[c * f1 + m] : 0.f;
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
          if (c0 >= fp0) break;
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = w0v[c0 + i];
          tmem_st16(tq + T_W0 + (uint32_t)(mb0 * fp0 + c0), v);
          st_shared_v4(w0t.saddr + w0t.off(m, c0), pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                       pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
          st_shared_v4(w0t.saddr + w0t.off(m, c0 + 8), pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]),
                       pack_bf16x2(v[12], v[13]), pack_bf16x2(v[14], v[15]));
        }
      }
    }
    for (int c = tid; c < f1 + f2 + f3; c += THREADS) {
      const int l = c < f1 ? 0 : (c < f1 + f2 ? 1 : 2);
      const int o = l == 0 ? c : (l == 1 ? c - f1 : c - f1 - f2);
      bias[c] = Ws[g.boff[l] + o];
    }
    for (int k = tid; k <= f3; k += THREADS) wh[k] = k < f3 ? Ws[g.woff[3] + k] : Ws[g.boff[3]];

    FS_PROF(26);
    const int64_t slot_words = ((int64_t)B * g.sum_hidden + 31) / 32;
    bool have_next = false;
    int cur = 0;  // s_rowidx_pp / s_y_pp buffer of the current chunk
    uint4 xnext[XPRE];
    MaskRaw mrn;
    uint32_t kw[4];   // keep words of this warp's forward items (current chunk)
    uint32_t kwn[4];  // the same for the prefetched next chunk (transposed in the stage-2 MMA shadow)
    // per-client constants, loaded once (the stores into W would otherwise
    // force the compiler to reload them every step)
    const int64_t row_off = a.row_off[rq];
    const int32_t* perm_c = a.perm + a.perm_off[rq];
    const uint32_t* mask_c = a.mask_mode == FS_MASK_BITS ? a.mask_bits + a.mask_off[rq] : nullptr;
    const double* lr_c = a.lr + (int64_t)rq * a.epochs;
    const int step_begin = a.start_step[rq], step_end = a.end_step[rq];
    float lr = step_begin < step_end ? (float)lr_c[step_begin / spe] : 0.f;

    for (int step = step_begin; step < step_end; ++step) {
      const int e = step / spe, s = step % spe;
      const int step_rows = min(B, n - s * B);
      const int32_t* perm_e = perm_c + (int64_t)e * n;
      const uint32_t* mbits = mask_c ? mask_c + (int64_t)step * slot_words : nullptr;
      const float dsc = mbits ? a.scale : 1.f;
      const int nchunks = (step_rows + R - 1) / R;

      for (int ch = 0; ch < nchunks; ++ch) {
        const int row0 = ch * R;
        const int rows = min(R, step_rows - row0);
        const bool last_chunk = ch == nchunks - 1;
        const bool first_chunk = ch == 0;
        // ---------------- gather the chunk's rows (bf16 features) and labels
        const int cpr = fp0 / 8;
        if (have_next) {  // staged during the previous chunk: row ids, labels, X rows, keep words
          cur ^= 1;
#pragma unroll
          for (int k = 0; k < 4; ++k) kw[k] = kwn[k];
        } else {
          if (tid < R) {
            const int64_t row = tid < rows ? row_off + perm_e[s * B + row0 + tid] : -1;
            s_rowidx_pp[cur][tid] = row;
            s_y_pp[cur][tid] = row >= 0 ? __ldcg(a.labels + row) : 0.f;
          }
          named_sync(THREADS);
        }
        FS_PROF(0);
        {
#pragma unroll
          for (int u = 0; u < XPRE; ++u) {
            const int i = tid + u * THREADS;
            if (i < R * cpr) {
              const int r = i / cpr, c = (i % cpr) * 8;
              uint4 v = xnext[u];
              if (!have_next) {
                v = make_uint4(0, 0, 0, 0);
                if (r < rows) v = __ldcg(reinterpret_cast<const uint4*>(a.feat + s_rowidx_pp[cur][r] * fp0 + c));
              }
              st_shared_v4(xt.saddr + xt.off(r, c), v.x, v.y, v.z, v.w);
            }
          }
        }
        FS_PROF(28);
        const int hh_w = warp >> 2;  // row half of this warp's forward items
        if (!have_next) {
          if (mbits && a.mask_flags) wait_mask_step(a.mask_flags + (int64_t)rq * a.max_steps + step, a.mask_tag);
          mask_issue(mrn, mbits, step_rows, row0, rows, f1, f2, f3, MB, q, hh_w, lane);
          mask_finish(mrn, mbits != nullptr, step_rows, rows, f1, f2, f3, MB, q, hh_w, lane, kw);
        }
        FS_PROF(29);
        have_next = false;
        int nstep = step, nch = ch + 1;
        if (nch == nchunks) {
          nstep = step + 1;
          nch = 0;
        }
        const bool next_ok = nstep < step_end;
        const int nsr = next_ok ? min(B, n - (nstep % spe) * B) : 0;  // next chunk: its step's rows
        const int nrows = next_ok ? min(R, nsr - nch * R) : 0;        // and its own rows

        // ---------------- F0: H1^T = relu(W0^T X^T + b0) * mask
        stage_sync();
        if (warp == 0) {
          const uint32_t id = idesc_bf16(128, R, false, false);
          for (int ks = 0; ks < fp0 / 16; ++ks)
            for (int mb = 0; mb < MB; ++mb)
              mma_bf16_ws(tbase + T_ACC + (uint32_t)(mb * R), w0t.kmajor(ks, mb), xt.kmajor(ks), id, ks > 0);
          mma_commit_ws(&mma_bar);
        }
        {
          wait_mma(&mma_bar, phase);
          FS_PROF(1);
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int it = warp + 8 * k;
            if (it >= MB * 8) break;
            const int hh = (it >> 2) & 1, mb = it >> 3;
            const int m = mb * 128 + q * 32 + lane;
            uint32_t raw[32];
            tmem_ld32_nw(tq + T_ACC + (uint32_t)(mb * R + hh * 32), raw);
            const uint32_t keep = kw[k];
            const float b = bias[m];
            tmem_wait_ld_r(raw);
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float x = fmaxf(__uint_as_float(raw[j]) + b, 0.f);
              v[j] = ((keep >> j) & 1u) ? x * dsc : 0.f;
            }
            store_row32(h1t, m, hh * 32, v);
          }
        }
        FS_PROF(5);

        // ---------------- F1: H2^T = relu(W1^T H1^T + b1) * mask
        stage_sync();
        if (warp == 0) {
          const uint32_t id = idesc_bf16(128, R, true, true);
          for (int ks = 0; ks < f1 / 16; ++ks) mma_bf16_ws(tbase + T_ACC, w1t.mnmajor(ks), h1t.mnmajor(ks), id, ks > 0);
          mma_commit_ws(&mma_bar);
        }
        {
          const int hh = warp >> 2, m = q * 32 + lane;
          wait_mma(&mma_bar, phase);
          FS_PROF(2);
          uint32_t raw[32];
          tmem_ld32_nw(tq + T_ACC + (uint32_t)(hh * 32), raw);
          const uint32_t keep = kw[2];
          const float b = bias[f1 + m];
          tmem_wait_ld_r(raw);
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float x = fmaxf(__uint_as_float(raw[j]) + b, 0.f);
            v[j] = ((keep >> j) & 1u) ? x * dsc : 0.f;
          }
          store_row32(h2t, m, hh * 32, v);
        }
        FS_PROF(6);

        // ---------------- F2: H3^T = relu(W2^T H2^T + b2) * mask, head logits
        stage_sync();
        if (warp == 0) {
          const uint32_t id = idesc_bf16(128, R, true, true);  // M = 128 over 64 units (upper half unused)
          for (int ks = 0; ks < f2 / 16; ++ks) mma_bf16_ws(tbase + T_ACC, w2t.mnmajor(ks), h2t.mnmajor(ks), id, ks > 0);
          mma_commit_ws(&mma_bar);
        }
        if (next_ok && tid >= 64 && tid < 64 + R) {
          // prefetch A: next chunk's row ids and labels, by warps 2-3, which
          // have no F2 output units (their dependent global loads overlap the F2 stage)
          const int t = tid - 64;
          const int ne = nstep / spe, ns = nstep % spe;
          const int nrows_step = min(B, n - ns * B);
          const int nr0 = nch * R;
          const int64_t row = t < min(R, nrows_step - nr0) ? row_off + perm_c[(int64_t)ne * n + ns * B + nr0 + t] : -1;
          s_rowidx_pp[cur ^ 1][t] = row;
          s_y_pp[cur ^ 1][t] = row >= 0 ? __ldcg(a.labels + row) : 0.f;
        }
        {
          const int hh = warp >> 2, m = q * 32 + lane;
          const bool act = q < f3 / 32;  // warp-uniform
          wait_mma(&mma_bar, phase);
          FS_PROF(3);
          if (act) {
            uint32_t raw[32];
            tmem_ld32_nw(tq + T_ACC + (uint32_t)(hh * 32), raw);
            const uint32_t keep = kw[3];
            const float b = bias[f1 + f2 + m];
            const float w = wh[m];
            tmem_wait_ld_r(raw);
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float x = fmaxf(__uint_as_float(raw[j]) + b, 0.f);
              v[j] = ((keep >> j) & 1u) ? x * dsc : 0.f;
            }
            store_row32(h3t, m, hh * 32, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= w;
            zpart[q * R + hh * 32 + lane] = reduce_scatter32(v, lane);
          }
        }
        FS_PROF(7);
        __syncthreads();
        // ---------------- head: dz = (sigmoid(z) - y) / step_rows
        if (tid < R) {
          const float z = zpart[tid] + zpart[R + tid] + wh[f3];
          float d = 0.f;
          if (tid < rows) {
            d = (bf16::sigmoidf_stable(z) - s_y_pp[cur][tid]) / (float)step_rows;
            if (!isfinite(z)) atomicOr(a.status + rq, 1);
          }
          dz_sh[tid] = d;
          float t = d;
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
          if (lane == 0) gbh[warp] = t;
        }
        __syncthreads();
        FS_PROF(9);
        if (next_ok) {  // next chunk's keep-bit words (transposed in the stage-2 MMA shadow)
          if (mask_c && a.mask_flags && nch == 0)
            wait_mask_step(a.mask_flags + (int64_t)rq * a.max_steps + nstep, a.mask_tag);
          mask_issue(mrn, mask_c ? mask_c + (int64_t)nstep * slot_words : nullptr, nsr, nch * R, nrows, f1, f2, f3,
                     MB, q, warp >> 2, lane);
        }
        if (next_ok) {  // prefetch B: next chunk's feature rows, held in registers
#pragma unroll
          for (int u = 0; u < XPRE; ++u) {
            const int i = tid + u * THREADS;
            xnext[u] = make_uint4(0, 0, 0, 0);
            if (i < R * cpr) {
              const int64_t row = s_rowidx_pp[cur ^ 1][i / cpr];
              if (row >= 0) xnext[u] = __ldcg(reinterpret_cast<const uint4*>(a.feat + row * fp0 + (i % cpr) * 8));
            }
          }
          have_next = true;
        }
#if FS_D3_QUARTERS
        // ---------------- D3^T = gate(w_h dz^T, H3^T) * scale; head-weight and b2 gradient partials.
        // Every warp takes a (32-unit group, 16-row quarter) item; the partials
        // go to [4][64] slots in the gb0p area (consumed by stage 2, rewritten
        // only in stage 1)
        if (warp < 4 * (f3 / 32)) {
          const int ug = warp % (f3 / 32), rq4 = warp / (f3 / 32), m = ug * 32 + lane, c0 = rq4 * 16;
          uint32_t hv[8];
          ld_shared_v4(h3t.saddr + h3t.off(m, c0), hv[0], hv[1], hv[2], hv[3]);
          ld_shared_v4(h3t.saddr + h3t.off(m, c0 + 8), hv[4], hv[5], hv[6], hv[7]);
          const float w = wh[m] * dsc;
          float d[16];
          float gw = 0.f, gb = 0.f;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float hj = (j & 1) ? bf16hi(hv[j >> 1]) : bf16lo(hv[j >> 1]);
            const float dzj = dz_sh[c0 + j];
            gw = fmaf(hj, dzj, gw);
            d[j] = hj > 0.f ? dzj * w : 0.f;
          }
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            pk[j >> 1] = pack_bf16x2(d[j], d[j + 1]);
            gb += bf16lo(pk[j >> 1]);
            gb += bf16hi(pk[j >> 1]);
          }
          st_shared_v4(h3t.saddr + h3t.off(m, c0), pk[0], pk[1], pk[2], pk[3]);
          st_shared_v4(h3t.saddr + h3t.off(m, c0 + 8), pk[4], pk[5], pk[6], pk[7]);
          gb0p[rq4 * 64 + m] = gw;
          gb0p[256 + rq4 * 64 + m] = gb;
        }
#else
        // ---------------- D3^T = gate(w_h dz^T, H3^T) * scale; head-weight and b2 gradient partials
        if (q < f3 / 32) {
          const int hh = warp >> 2, m = q * 32 + lane;
          uint32_t hv[16];
          load_row32(h3t, m, hh * 32, hv);
          const float w = wh[m] * dsc;
          float d[32];
          float gw = 0.f, gb = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float hj = bf16_at(hv, j);
            const float dzj = dz_sh[hh * 32 + j];
            gw = fmaf(hj, dzj, gw);
            d[j] = hj > 0.f ? dzj * w : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const uint32_t p = pack_bf16x2(d[j], d[j + 1]);
            gb += bf16lo(p);
            gb += bf16hi(p);
          }
          store_row32(h3t, m, hh * 32, d);
          gwp[hh * 64 + m] = gw;
          gb2p[hh * 64 + m] = gb;
        }
#endif
        FS_PROF(11);

        // ---------------- stage 2: G2 = H2^T D3 (TMEM [0,64)), D2^T = W2 D3^T (TMEM [64,128))
        stage_sync();
        if (warp == 7) {  // stage 2 issued by warp 7: warp 0 transposes keep words in its shadow
          const uint32_t idg = idesc_bf16(128, f3, false, false);
          for (int ks = 0; ks < R / 16; ++ks) mma_bf16_ws(tbase + T_ACC, h2t.kmajor(ks), h3t.kmajor(ks), idg, ks > 0);
          const uint32_t idd = idesc_bf16(128, R, false, true);
          for (int ks = 0; ks < f3 / 16; ++ks) mma_bf16_ws(tbase + T_D2, w2t.kmajor(ks), h3t.mnmajor(ks), idd, ks > 0);
          mma_commit_ws(&mma_bar);
        }
        // head and b2 updates while the MMAs run (gradients accumulate over a step's chunks)
        if (tid >= 32 && tid <= 32 + f3) {
          const int k = tid - 32;
#if FS_D3_QUARTERS
          const float gk = k < f3 ? (gb0p[k] + gb0p[64 + k]) + (gb0p[128 + k] + gb0p[192 + k]) : gbh[0] + gbh[1];
#else
          const float gk = k < f3 ? gwp[k] + gwp[64 + k] : gbh[0] + gbh[1];
#endif
          const float acc = first_chunk ? gk : ghs[k] + gk;
          if (last_chunk) wh[k] -= lr * acc; else ghs[k] = acc;
        } else if (tid >= 128 && tid < 128 + f3) {
          const int c = tid - 128;
#if FS_D3_QUARTERS
          const float gk = (gb0p[256 + c] + gb0p[320 + c]) + (gb0p[384 + c] + gb0p[448 + c]);
#else
          const float gk = gb2p[c] + gb2p[64 + c];
#endif
          const float acc = first_chunk ? gk : gbacc[f1 + f2 + c] + gk;
          if (last_chunk) bias[f1 + f2 + c] -= lr * acc; else gbacc[f1 + f2 + c] = acc;
        }
        // the next chunk's keep words, off the chunk-start path
        if (next_ok && warp != 7) mask_finish(mrn, mask_c != nullptr, nsr, nrows, f1, f2, f3, MB, q, warp >> 2, lane, kwn);
        wait_mma(&mma_bar, phase);
        FS_PROF(14);
        {
          const int hh = warp >> 2, m = q * 32 + lane;
          // D2 carries the step size from here on: tiles hold -lr * dL/dH
          gb1p[hh * 128 + m] = gate_seg(h2t, m, hh * 32, tq + T_D2 + (uint32_t)(hh * 32), -lr * dsc);
        }
        // G2 (unit m = row of W2, columns [32hh, 32hh+32)) into registers; the
        // W2 update itself runs in the shadow of the stage-1 MMAs
        float gv[32];
        tmem_ld32(tq + T_ACC + (uint32_t)((warp >> 2) * 32), gv);
        FS_PROF(18);

        // ---------------- stage 1: W1 master += H1^T D2 (TMEM), D1^T = W1 D2^T (TMEM [0, MB*64))
        stage_sync();
        if (warp == 0) {
          const uint32_t idg = idesc_bf16(128, f2, false, false);
          for (int mb = 0; mb < MB; ++mb)
            for (int ks = 0; ks < R / 16; ++ks)
              mma_bf16_ws(tbase + T_W1 + (uint32_t)(mb * f2), h1t.kmajor(ks, mb), h2t.kmajor(ks), idg, 1u);
          const uint32_t idd = idesc_bf16(128, R, false, true);
          for (int mb = 0; mb < MB; ++mb)
            for (int ks = 0; ks < f2 / 16; ++ks)
              mma_bf16_ws(tbase + T_ACC + (uint32_t)(mb * R), w1t.kmajor(ks, mb), h2t.mnmajor(ks), idd, ks > 0);
          mma_commit_ws(&mma_bar);
        }
        if (tid >= 128 && tid < 128 + f2) {  // b1 += sum(-lr D2)
          const int c = tid - 128;
          const float gk = gb1p[c] + gb1p[128 + c];
          const float acc = first_chunk ? gk : gbacc[f1 + c] + gk;
          if (last_chunk) bias[f1 + c] += acc; else gbacc[f1 + c] = acc;
        }
        {  // W2 -= lr * G2 on the shared-memory master; bf16 tile after the step's last chunk
          const int hh = warp >> 2, m = q * 32 + lane;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float* p = w2m + (hh * 32 + j) * f2 + m;
            const float nw = *p - lr * gv[j];
            *p = nw;
            gv[j] = nw;
          }
          if (last_chunk) store_row32(w2t, m, hh * 32, gv);
        }
        if (next_ok && warp == 7) mask_finish(mrn, mask_c != nullptr, nsr, nrows, f1, f2, f3, MB, q, warp >> 2, lane, kwn);
        wait_mma(&mma_bar, phase);
        FS_PROF(13);
        for (int it = warp; it < MB * 8; it += 8) {
          const int hh = (it >> 2) & 1, mb = it >> 3;
          const int m = mb * 128 + q * 32 + lane;
          gb0p[hh * 256 + m] = gate_seg(h1t, m, hh * 32, tq + T_ACC + (uint32_t)(mb * R + hh * 32), dsc);
        }
        FS_PROF(17);

        // ---------------- stage 0: W0^T master += D1^T X (TMEM)
        stage_sync();
        if (warp == 0) {
          const uint32_t idg = idesc_bf16(128, fp0, false, true);
          for (int mb = 0; mb < MB; ++mb)
            for (int ks = 0; ks < R / 16; ++ks)
              mma_bf16_ws(tbase + T_W0 + (uint32_t)(mb * fp0), h1t.kmajor(ks, mb), xt.mnmajor(ks), idg, 1u);
          mma_commit_ws(&mma_bar);
        }
        if (tid < f1) {  // b0 += sum(-lr D1)
          const float gk = gb0p[tid] + gb0p[256 + tid];
          const float acc = first_chunk ? gk : gbacc[tid] + gk;
          if (last_chunk) bias[tid] += acc; else gbacc[tid] = acc;
        }
        if (last_chunk) {  // refresh the bf16 W1 tile from the TMEM master (stage 1's MMAs are done with it)
          for (int it = warp; it < MB * 8; it += 8) {
            const int hh = (it >> 2) & 1, mb = it >> 3;
            const int m = mb * 128 + q * 32 + lane;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int c0 = hh * (f2 / 2) + 32 * k;
              float v[32];
              tmem_ld32(tq + T_W1 + (uint32_t)(mb * f2 + c0), v);
              store_row32(w1t, m, c0, v);
            }
          }
        }
        wait_mma(&mma_bar, phase);
        FS_PROF(12);
        if (last_chunk) {  // refresh the bf16 W0^T tile from the TMEM master
          for (int it = warp; it < MB * 4; it += 8) {
            const int mb = it >> 2;
            const int m = mb * 128 + q * 32 + lane;
            for (int c0 = 0; c0 < fp0; c0 += 16) {
              float v[16];
              tmem_ld16(tq + T_W0 + (uint32_t)(mb * fp0 + c0), v);
              st_shared_v4(w0t.saddr + w0t.off(m, c0), pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                           pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
              st_shared_v4(w0t.saddr + w0t.off(m, c0 + 8), pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]),
                           pack_bf16x2(v[12], v[13]), pack_bf16x2(v[14], v[15]));
            }
          }
        }
        FS_PROF(20);
        __syncthreads();
        FS_PROF(25);
      }  // chunks
      if ((step + 1) % spe == 0 && step + 1 < step_end) lr = (float)lr_c[(step + 1) / spe];
    }    // steps

    // ---------------- client end: write the trained row once
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    FS_PROF(27);
    for (int it = warp; it < MB * 4; it += 8) {  // W_0 (row-major [f0 x f1]) from the W_0^T master
      const int mb = it >> 2;
      const int m = mb * 128 + q * 32 + lane;
      for (int c0 = 0; c0 < fp0; c0 += 16) {
        float v[16];
        tmem_ld16(tq + T_W0 + (uint32_t)(mb * fp0 + c0), v);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c0 + i < f0) W[(c0 + i) * f1 + m] = v[i];
      }
    }
    for (int it = warp; it < MB * 8; it += 8) {  // W_1
      const int hh = (it >> 2) & 1, mb = it >> 3;
      const int m = mb * 128 + q * 32 + lane;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int c0 = hh * (f2 / 2) + 32 * k;
        float v[32];
        tmem_ld32(tq + T_W1 + (uint32_t)(mb * f2 + c0), v);
        float* dst = W + g.woff[1] + (int64_t)m * f2 + c0;
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    }
    {  // W_2 rows from the column-major master (conflict-free smem reads, 16-byte stores)
      const int hh = warp >> 2, m = q * 32 + lane;
      float* dst = W + g.woff[2] + (int64_t)m * f3 + hh * 32;
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4*>(dst + i) = make_float4(w2m[(hh * 32 + i) * f2 + m], w2m[(hh * 32 + i + 1) * f2 + m],
                                                          w2m[(hh * 32 + i + 2) * f2 + m],
                                                          w2m[(hh * 32 + i + 3) * f2 + m]);
    }
    for (int c = tid; c < f1 + f2 + f3; c += THREADS) {
      const int l = c < f1 ? 0 : (c < f1 + f2 ? 1 : 2);
      const int o = l == 0 ? c : (l == 1 ? c - f1 : c - f1 - f2);
      W[g.boff[l] + o] = bias[c];
    }
    for (int k = tid; k <= f3; k += THREADS) {
      if (k < f3) W[g.woff[3] + k] = wh[k]; else W[g.boff[3]] = wh[f3];
    }
    if (a.done || a.counts_out) {  // fused K6 count (+ release of the completion record)
      __threadfence();
      __syncthreads();
      client_done(g.M, a.align_mode, W, Ws,
                  a.align_mode == FS_ALIGN_DELTA_SIGN ? reinterpret_cast<const float*>(a.w_prev[rq]) : nullptr,
                  a.status + rq, a.done ? a.done[rq] : 0, a.done_tag, tid,
                  a.counts_out ? a.counts_out + rq : nullptr);
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
  }
  fence_before_sync();
  __syncthreads();
  if (a.prof && tid < 32) atomicAdd(a.prof + tid, s_prof[tid]);
  if (warp == 0) tmem_dealloc(tbase, bf16::TMEM_COLS);
}

// ---------------------------------------------------------------------------
// K8 forward (bf16 mode): class-1 probabilities of the test rows under the
// fp32 global model, same unit-major tcgen05 forward as the trainer (bf16
// operands, fp32 accumulation, fp32 head/sigmoid), one 64-row chunk per CTA
// iteration. The fp64 parity mode keeps fs_forward_f64.
struct EvalLay {
  uint32_t x, h1, h2, w0, w1, w2, pad, fl, total;
};
__host__ __device__ inline EvalLay eval_lay(const Geo& g) {
  EvalLay l;
  uint32_t s = 0;
  l.x = s;   s += (uint32_t)(R * g.fp[0] * 2);
  l.h1 = s;  s += (uint32_t)(g.f[1] * R * 2);
  l.h2 = s;  s += (uint32_t)(g.f[2] * R * 2);
  l.w0 = s;  s += (uint32_t)(g.f[1] * g.fp[0] * 2);
  l.w1 = s;  s += (uint32_t)(g.f[1] * g.f[2] * 2);
  l.w2 = s;  s += (uint32_t)(g.f[2] * g.f[3] * 2);
  l.pad = s; s += 16 * 1024;  // F2 (M = 128 over 64 units) reads past the W_2 tile
  l.fl = s;  s += (uint32_t)((g.f[1] + g.f[2] + g.f[3] + g.f[3] + 1 + 2 * R) * 4);
  l.total = s;
  return l;
}

__global__ void __launch_bounds__(THREADS, 1) eval_kernel(Geo g, const float* __restrict__ w,
                                                       const __nv_bfloat16* __restrict__ xb, int n,
                                                       double* __restrict__ probs) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mma_bar;
  __shared__ uint32_t tmem_base_sh;
  const EvalLay ly = eval_lay(g);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = warp & 3;
  const int f0 = g.f[0], fp0 = g.fp[0], f1 = g.f[1], f2 = g.f[2], f3 = g.f[3];
  const int MB = f1 / 128;
  float* fl = reinterpret_cast<float*>(smem + ly.fl);
  float* bias = fl;                         // [f1 + f2 + f3]
  float* wh = fl + f1 + f2 + f3;            // [f3 + 1]
  float* zpart = wh + f3 + 1;               // [2][R]
  const Tile xt{smem_u32(smem + ly.x), R};
  const Tile h1t{smem_u32(smem + ly.h1), f1};
  const Tile h2t{smem_u32(smem + ly.h2), f2};
  const Tile w0t{smem_u32(smem + ly.w0), f1};
  const Tile w1t{smem_u32(smem + ly.w1), f1};
  const Tile w2t{smem_u32(smem + ly.w2), f2};

  if (warp == 0) tmem_alloc(&tmem_base_sh, 128);
  if (tid == 0) {
    mbar_init(&mma_bar, 1);
    fence_mbar_init();
  }
  // weights: bf16 tiles (unit-major W_0^T) and fp32 biases / head
  for (int i = tid; i < f1 * (fp0 / 8); i += THREADS) {
    const int m = i % f1, c0 = (i / f1) * 8;
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = c0 + k < f0 ? w[(c0 + k) * f1 + m] : 0.f;
    st_shared_v4(w0t.saddr + w0t.off(m, c0), pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                 pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
  }
  for (int i = tid; i < f1 * (f2 / 8); i += THREADS) {
    const int m = i / (f2 / 8), c0 = (i % (f2 / 8)) * 8;
    const float* src = w + g.woff[1] + (int64_t)m * f2 + c0;
    st_shared_v4(w1t.saddr + w1t.off(m, c0), pack_bf16x2(src[0], src[1]), pack_bf16x2(src[2], src[3]),
                 pack_bf16x2(src[4], src[5]), pack_bf16x2(src[6], src[7]));
  }
  for (int i = tid; i < f2 * (f3 / 8); i += THREADS) {
    const int m = i / (f3 / 8), c0 = (i % (f3 / 8)) * 8;
    const float* src = w + g.woff[2] + (int64_t)m * f3 + c0;
    st_shared_v4(w2t.saddr + w2t.off(m, c0), pack_bf16x2(src[0], src[1]), pack_bf16x2(src[2], src[3]),
                 pack_bf16x2(src[4], src[5]), pack_bf16x2(src[6], src[7]));
  }
  for (int c = tid; c < f1 + f2 + f3; c += THREADS) {
    const int l = c < f1 ? 0 : (c < f1 + f2 ? 1 : 2);
    const int o = l == 0 ? c : (l == 1 ? c - f1 : c - f1 - f2);
    bias[c] = w[g.boff[l] + o];
  }
  for (int k = tid; k <= f3; k += THREADS) wh[k] = k < f3 ? w[g.woff[3] + k] : w[g.boff[3]];
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = tmem_base_sh;
  const uint32_t tq = tbase + ((uint32_t)(q * 32) << 16);
  uint32_t phase = 0;
  const int cpr = fp0 / 8;
  const int nchunks = (n + R - 1) / R;

  for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int r0 = ch * R;
    const int rows = min(R, n - r0);
    for (int i = tid; i < R * cpr; i += THREADS) {
      const int r = i / cpr, c = (i % cpr) * 8;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < rows) v = __ldg(reinterpret_cast<const uint4*>(xb + (int64_t)(r0 + r) * fp0 + c));
      st_shared_v4(xt.saddr + xt.off(r, c), v.x, v.y, v.z, v.w);
    }
    // F0
    stage_sync();
    if (warp == 0) {
      const uint32_t id = idesc_bf16(128, R, false, false);
      for (int ks = 0; ks < fp0 / 16; ++ks)
        for (int mb = 0; mb < MB; ++mb)
          mma_bf16_ws(tbase + (uint32_t)(mb * R), w0t.kmajor(ks, mb), xt.kmajor(ks), id, ks > 0);
      mma_commit_ws(&mma_bar);
    }
    wait_mma(&mma_bar, phase);
    for (int it = warp; it < MB * 8; it += 8) {
      const int hh = (it >> 2) & 1, mb = it >> 3;
      const int m = mb * 128 + q * 32 + lane;
      float v[32];
      tmem_ld32(tq + (uint32_t)(mb * R + hh * 32), v);
      const float b = bias[m];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j] + b, 0.f);
      store_row32(h1t, m, hh * 32, v);
    }
    // F1
    stage_sync();
    if (warp == 0) {
      const uint32_t id = idesc_bf16(128, R, true, true);
      for (int ks = 0; ks < f1 / 16; ++ks) mma_bf16_ws(tbase, w1t.mnmajor(ks), h1t.mnmajor(ks), id, ks > 0);
      mma_commit_ws(&mma_bar);
    }
    wait_mma(&mma_bar, phase);
    {
      const int hh = warp >> 2, m = q * 32 + lane;
      float v[32];
      tmem_ld32(tq + (uint32_t)(hh * 32), v);
      const float b = bias[f1 + m];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j] + b, 0.f);
      store_row32(h2t, m, hh * 32, v);
    }
    // F2 + head
    stage_sync();
    if (warp == 0) {
      const uint32_t id = idesc_bf16(128, R, true, true);
      for (int ks = 0; ks < f2 / 16; ++ks) mma_bf16_ws(tbase, w2t.mnmajor(ks), h2t.mnmajor(ks), id, ks > 0);
      mma_commit_ws(&mma_bar);
    }
    wait_mma(&mma_bar, phase);
    if (q < f3 / 32) {
      const int hh = warp >> 2, m = q * 32 + lane;
      float v[32];
      tmem_ld32(tq + (uint32_t)(hh * 32), v);
      const float b = bias[f1 + f2 + m], wm = wh[m];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j] + b, 0.f) * wm;
      zpart[q * R + hh * 32 + lane] = reduce_scatter32(v, lane);
    }
    __syncthreads();
    if (tid < rows) probs[r0 + tid] = (double)bf16::sigmoidf_stable(zpart[tid] + zpart[R + tid] + wh[f3]);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 128);
}

int launch_eval(const Geo& g, const float* w, const void* xb, int n, double* probs, cudaStream_t st) {
  const uint32_t bytes = eval_lay(g).total;
  ensure_smem(eval_kernel, (int)bytes);
  const int chunks = (n + R - 1) / R;
  const int grid = chunks < kNumSMs ? chunks : kNumSMs;
  eval_kernel<<<grid, THREADS, bytes, st>>>(g, w, reinterpret_cast<const __nv_bfloat16*>(xb), n, probs);
  return check_launch("bf16t::eval_kernel");
}

int launch(const Args& a, int grid, cudaStream_t st) {
  const uint32_t bytes = lay_of(a.g).total;
  ensure_smem(train_kernel, (int)bytes);
  train_kernel<<<grid, THREADS, bytes, st>>>(a);
  return check_launch("bf16t::train_kernel");
}

}  // namespace bf16t
}  // namespace fs
