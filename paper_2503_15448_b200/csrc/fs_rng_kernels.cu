// K1-K3: per-round randomness of the round loop, generated on device.
//
//   K1 fs_train_seeds    derive_seed(master, "train", cid, cycle)  server.py:207
//   K2 fs_shuffle_perms  derive_rng(seed, "shuffle", e).permutation(n)  client.py:136
//   K3 fs_dropout_bits   dropout_masks(spec, b, derive_seed(seed, "mask", e, s))
//                        model.py:153-166, client.py:150
//
// All three are integer work (SeedSequence uint32 hashing, PCG64 128-bit LCG
// steps); outputs are bit-exact with numpy's streams (fs_rng.cuh).
#include "fs_common.cuh"
#include "fs_rng.cuh"

#include <cmath>
#include <cstdlib>

namespace fs {

__global__ void train_seeds_kernel(uint64_t master, const int32_t* cid, const int32_t* cyc, int n,
                                   uint64_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = derive_train_seed(master, (uint32_t)cid[i], (uint32_t)cyc[i]);
}

// One CTA per (request, epoch): Fisher-Yates over random_interval draws.
// The draw chain is inherently sequential (rejection sampling on a buffered
// 32-bit stream), so one lane runs it while the array lives in shared
// memory (or in the output itself for shards too large to stage).
__global__ void shuffle_kernel(const uint64_t* seeds, const int32_t* n_rows, const int64_t* perm_off,
                               int epochs, int32_t* perm_out, int use_smem) {
  extern __shared__ int32_t sh_perm[];
  const int r = blockIdx.x / epochs, e = blockIdx.x % epochs;
  const int n = n_rows[r];
  int32_t* out = perm_out + perm_off[r] + (int64_t)e * n;
  int32_t* a = use_smem ? sh_perm : out;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = i;
  __syncthreads();
  if (threadIdx.x == 0) {
    Pcg64 g = pcg_shuffle_stream(seeds[r], (uint32_t)e);
    for (int i = n - 1; i > 0; --i) {
      const int j = (int)g.interval((uint64_t)i);
      const int32_t t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
  }
  __syncthreads();
  if (use_smem)
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = a[i];
}

constexpr int MASK_THREADS = 128;
constexpr int MASK_YSPLIT = 8;
constexpr int MASK_ILP = 4;  // independent PCG64 sub-streams per thread

// LCG jump by k steps, independent of the stream: state' = a*state + g*inc.
struct LcgJump {
  U128 a, g;
};
FS_HD LcgJump lcg_jump(uint64_t k) {
  U128 acc_mult{0, 1}, acc_plus{0, 0};
  U128 cur_mult = pcg_mult(), cur_plus{0, 1};
  const U128 one{0, 1};
  while (k) {
    if (k & 1) {
      acc_mult = u128_mul(acc_mult, cur_mult);
      acc_plus = u128_add(u128_mul(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = u128_mul(u128_add(cur_mult, one), cur_plus);
    cur_mult = u128_mul(cur_mult, cur_mult);
    k >>= 1;
  }
  return LcgJump{acc_mult, acc_plus};
}
__device__ __forceinline__ U128 lcg_apply(const LcgJump& j, U128 state, U128 inc) {
  return u128_add(u128_mul(j.a, state), u128_mul(j.g, inc));
}
__device__ __forceinline__ uint64_t xsl_rr(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// Packs keep-bits of one stream: bit j = (random_j < keep), with
// random() = (x >> 11) * 2^-53 < keep  <=>  (x >> 11) < ceil(keep * 2^53)
// (integer comparison, threshold computed exactly on host). Thread t owns
// words t, t + T, t + 2T, ... (T = MASK_THREADS) and runs MASK_ILP of them
// at once as independent LCG chains: word w starts 32w steps after `base`,
// reached with precomputed jumps (jt: 32t steps, j1: 32T steps, jr: from the
// end of a word to the thread's word MASK_ILP*T further on).
// One PCG64 step on 32-bit limbs: state = state * MULT + inc (mod 2^128),
// the 128-bit additions as add.cc/addc carry chains (the C++ form spends its
// ALU slots on compare-and-select carries; K3 is ALU-pipe bound).
__device__ __forceinline__ void lcg128_step(uint64_t& hi, uint64_t& lo, uint64_t inc_hi, uint64_t inc_lo) {
  constexpr uint64_t M_LO = 0x4385DF649FCCF645ull, M_HI = 0x2360ED051FC65DA4ull;
  const uint64_t p_lo = lo * M_LO;
  const uint64_t p_hi = __umul64hi(lo, M_LO) + lo * M_HI + hi * M_LO;
  uint32_t r0, r1, r2, r3;
  asm("add.cc.u32 %0, %4, %8;\n\t"
      "addc.cc.u32 %1, %5, %9;\n\t"
      "addc.cc.u32 %2, %6, %10;\n\t"
      "addc.u32 %3, %7, %11;"
      : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
      : "r"((uint32_t)p_lo), "r"((uint32_t)(p_lo >> 32)), "r"((uint32_t)p_hi), "r"((uint32_t)(p_hi >> 32)),
        "r"((uint32_t)inc_lo), "r"((uint32_t)(inc_lo >> 32)), "r"((uint32_t)inc_hi), "r"((uint32_t)(inc_hi >> 32)));
  lo = ((uint64_t)r1 << 32) | r0;
  hi = ((uint64_t)r3 << 32) | r2;
}

// keep bit of the draw at the current state: XSL-RR output x, random() =
// (x >> 11) * 2^-53 < keep  <=>  x < thresh << 11 (thresh < 2^53). The 64-bit
// rotation is two 32-bit funnel shifts.
__device__ __forceinline__ uint32_t keep_of(uint64_t hi, uint64_t lo, uint32_t t_hi, uint32_t t_lo) {
  const uint64_t x = hi ^ lo;
  const uint32_t rot = (uint32_t)(hi >> 58);
  uint32_t a = (uint32_t)x, b = (uint32_t)(x >> 32);
  if (rot & 32) {
    const uint32_t t = a;
    a = b;
    b = t;
  }
  const uint32_t o_lo = __funnelshift_r(a, b, rot);
  const uint32_t o_hi = __funnelshift_r(b, a, rot);
  return (o_hi < t_hi || (o_hi == t_hi && o_lo < t_lo)) ? 1u : 0u;
}

// Packs keep-bits of one stream: bit j = (random_j < keep), with
// random() = (x >> 11) * 2^-53 < keep  <=>  (x >> 11) < ceil(keep * 2^53)
// (integer comparison, threshold computed exactly on host). Thread t owns
// words t, t + T, t + 2T, ... (T = MASK_THREADS) and runs MASK_ILP of them
// at once as independent LCG chains: word w starts 32w steps after `base`,
// reached with precomputed jumps (jt: 32t steps, j1: 32T steps, jr: from the
// end of a word to the thread's word MASK_ILP*T further on).
__device__ void mask_stream(U128 base_state, U128 inc, int64_t n_draws, uint64_t thresh, uint32_t* out,
                            const LcgJump& jt, const LcgJump& j1, const LcgJump& jr) {
  const int64_t words = (n_draws + 31) / 32;
  const int t = threadIdx.x;
  if (t >= words) return;
  const uint64_t tq = thresh << 11;
  const uint32_t t_hi = (uint32_t)(tq >> 32), t_lo = (uint32_t)tq;
  U128 s[MASK_ILP];
  s[0] = lcg_apply(jt, base_state, inc);
#pragma unroll
  for (int u = 1; u < MASK_ILP; ++u) s[u] = lcg_apply(j1, s[u - 1], inc);
  for (int64_t w = t; w < words; w += (int64_t)MASK_ILP * MASK_THREADS) {
    uint32_t bits[MASK_ILP];
#pragma unroll
    for (int u = 0; u < MASK_ILP; ++u) bits[u] = 0;
#pragma unroll 4
    for (int b = 0; b < 32; ++b) {
#pragma unroll
      for (int u = 0; u < MASK_ILP; ++u) {
        lcg128_step(s[u].hi, s[u].lo, inc.hi, inc.lo);
        // shift in from the top: after 32 draws bit j holds draw j
        bits[u] = __funnelshift_r(bits[u], keep_of(s[u].hi, s[u].lo, t_hi, t_lo), 1);
      }
    }
#pragma unroll
    for (int u = 0; u < MASK_ILP; ++u) {
      const int64_t wu = w + (int64_t)u * MASK_THREADS;
      if (wu < words) {
        const int64_t lim = n_draws - wu * 32;
        out[wu] = lim >= 32 ? bits[u] : (bits[u] & ((1u << lim) - 1u));
      }
      s[u] = lcg_apply(jr, s[u], inc);
    }
  }
}

// grid (request, MASK_YSPLIT): block y handles steps y, y + YSPLIT, ... of its
// request. Warp 0 derives up to 32 step streams at once (one lane each:
// SeedSequence hashing + PCG64 seeding), then all threads fill their words.
// K2 for shards of up to 65536 rows: one CTA of SH_THREADS per (request,
// epoch). The 32-bit draw stream (numpy's buffered next_uint32: low then high
// half of each PCG64 output) is generated SH_VB values at a time by all
// threads from LCG jumps; one thread then runs the sequential part alone:
// random_interval's masked rejection over the buffered values and the
// Fisher-Yates swaps on a 16-bit index array in shared memory (the next value
// is loaded ahead of each swap, so a step costs one shared-memory round trip
// instead of a 128-bit LCG step). Small footprint (2 KB + 2 bytes per row) so
// these CTAs fit beside the trainer's persistent CTAs.
constexpr int SH_THREADS = 64;
constexpr int SH_VB = 512;                       // draws per generated batch
constexpr int SH_M = SH_VB / 2 / SH_THREADS;     // PCG64 outputs per thread per batch
__global__ void __launch_bounds__(SH_THREADS)
    shuffle16_kernel(const uint64_t* seeds, const int32_t* n_rows, const int64_t* perm_off, int epochs,
                     int32_t* perm_out) {
  extern __shared__ __align__(16) uint8_t sh_raw[];
  uint32_t* vbuf = reinterpret_cast<uint32_t*>(sh_raw);     // [SH_VB]
  uint16_t* a = reinterpret_cast<uint16_t*>(vbuf + SH_VB);  // [n]
  __shared__ U128 sh_state, sh_inc;
  __shared__ int sh_i;
  const int tid = threadIdx.x;
  const int r = blockIdx.x / epochs, e = blockIdx.x % epochs;
  const int n = n_rows[r];
  int32_t* out = perm_out + perm_off[r] + (int64_t)e * n;
  for (int i = tid; i < n; i += SH_THREADS) a[i] = (uint16_t)i;
  if (tid == 0) {
    const Pcg64 g = pcg_shuffle_stream(seeds[r], (uint32_t)e);
    sh_state = g.state;
    sh_inc = g.inc;
  }
  const LcgJump j_init = lcg_jump((uint64_t)tid * SH_M);   // this thread's first output of a batch
  const LcgJump j_next = lcg_jump(SH_VB / 2 - SH_M);        // from its last output to the next batch
  __syncthreads();
  const U128 inc = sh_inc;
  U128 st = lcg_apply(j_init, sh_state, inc);
  int i = n - 1;  // Fisher-Yates position (thread 0)
  while (n > 1) {
#pragma unroll
    for (int j = 0; j < SH_M; ++j) {
      lcg128_step(st.hi, st.lo, inc.hi, inc.lo);
      const uint64_t x = xsl_rr(st);
      const int k = 2 * (tid * SH_M + j);
      vbuf[k] = (uint32_t)x;
      vbuf[k + 1] = (uint32_t)(x >> 32);
    }
    st = lcg_apply(j_next, st, inc);
    __syncthreads();
    if (tid == 0) {
      uint32_t vn = vbuf[0];
      for (int c = 1;; ++c) {
        const uint32_t v = vn & (0xFFFFFFFFu >> __clz(i));  // random_interval(i): smallest 2^k-1 >= i
        if (c < SH_VB) vn = vbuf[c];
        if (v <= (uint32_t)i) {
          const uint16_t ai = a[i], av = a[v];
          a[i] = av;
          a[v] = ai;
          if (--i == 0) break;
        }
        if (c == SH_VB) break;
      }
      sh_i = i;
    }
    __syncthreads();
    if (sh_i == 0) break;
  }
  __syncthreads();
  for (int k = tid; k < n; k += SH_THREADS) out[k] = a[k];
}

__global__ void __launch_bounds__(MASK_THREADS)
    dropout_bits_kernel(const uint64_t* seeds, const int32_t* n_rows, const int32_t* batch,
                        const int64_t* mask_off, int n_req, int epochs, int sum_hidden, uint64_t thresh,
                        uint32_t* bits) {
  // work item = (request, y-split); a throttled launch (fewer CTAs than items)
  // strides over them, so the mask generation can be given a bounded share
  // of the SMs it shares with the trainer and the round's tail kernels
  __shared__ U128 sh_state[32], sh_inc[32];
  const LcgJump jt = lcg_jump(32ull * threadIdx.x);
  const LcgJump j1 = lcg_jump(32ull * MASK_THREADS);
  const LcgJump jr = lcg_jump(32ull * MASK_THREADS * MASK_ILP - 32);
  for (int item = blockIdx.x; item < n_req * MASK_YSPLIT; item += gridDim.x) {
    const int r = item / MASK_YSPLIT, ysplit = item % MASK_YSPLIT;
    const int n = n_rows[r], B = batch[r];
    const int spe = (n + B - 1) / B;
    const int total = epochs * spe;
    const int64_t slot = ((int64_t)B * sum_hidden + 31) / 32;
    const uint64_t train_seed = seeds[r];
    uint32_t* out_r = bits + mask_off[r];
    for (int k0 = 0;; k0 += 32) {
      const int st0 = ysplit + k0 * MASK_YSPLIT;
      if (st0 >= total) break;
      __syncthreads();
      if (threadIdx.x < 32) {
        const int st = st0 + threadIdx.x * MASK_YSPLIT;
        if (st < total) {
          const Pcg64 g = pcg_from_seed(derive_mask_seed(train_seed, (uint32_t)(st / spe), (uint32_t)(st % spe)));
          sh_state[threadIdx.x] = g.state;
          sh_inc[threadIdx.x] = g.inc;
        }
      }
      __syncthreads();
      for (int j = 0; j < 32; ++j) {
        const int st = st0 + j * MASK_YSPLIT;
        if (st >= total) break;
        const int rows = min(B, n - (st % spe) * B);
        mask_stream(sh_state[j], sh_inc[j], (int64_t)rows * sum_hidden, thresh, out_r + (int64_t)st * slot, jt, j1,
                    jr);
      }
    }
  }
}

__global__ void __launch_bounds__(MASK_THREADS)
    dropout_bits_seed_kernel(uint64_t mask_seed, int64_t n_draws, uint64_t thresh, uint32_t* bits) {
  const Pcg64 g = pcg_from_seed(mask_seed);
  mask_stream(g.state, g.inc, n_draws, thresh, bits, lcg_jump(32ull * threadIdx.x), lcg_jump(32ull * MASK_THREADS),
              lcg_jump(32ull * MASK_THREADS * MASK_ILP - 32));
}

// K3, flagged: the keep bits of one (request, step) per CTA, dispatched
// step-major in the trainer's client order (block b -> step b / n, client
// order[b % n]), each step published with a release store of `tag` into
// flags[r * max_steps + step]. The trainer of the same round runs
// concurrently and waits per step on the flag (fs_train_desc.mask_flags), so
// the mask generation overlaps its own round's trainer instead of the
// previous round's tail. Per-thread LCG jumps are computed in the kernel (no
// host-side table copy, which as a synchronous cudaMemcpyToSymbol could wait
// behind a trainer that is itself waiting for these flags).

__global__ void __launch_bounds__(MASK_THREADS)
    dropout_bits_step_kernel(const uint64_t* seeds, const int32_t* n_rows, const int32_t* batch,
                             const int64_t* mask_off, const int32_t* order, int n_req, int epochs, int max_steps,
                             int sum_hidden, uint64_t thresh, uint32_t* bits, int32_t* flags, int32_t tag) {
  __shared__ U128 sh_state, sh_inc;
  const int b = blockIdx.x;
  const int st = b / n_req;
  const int r = order[b % n_req];
  const int n = n_rows[r], B = batch[r];
  const int spe = (n + B - 1) / B;
  if (st >= epochs * spe) return;
  if (threadIdx.x == 0) {
    const Pcg64 g = pcg_from_seed(derive_mask_seed(seeds[r], (uint32_t)(st / spe), (uint32_t)(st % spe)));
    sh_state = g.state;
    sh_inc = g.inc;
  }
  __syncthreads();
  const int64_t slot = ((int64_t)B * sum_hidden + 31) / 32;
  const int rows = min(B, n - (st % spe) * B);
  mask_stream(sh_state, sh_inc, (int64_t)rows * sum_hidden, thresh, bits + mask_off[r] + (int64_t)st * slot,
              lcg_jump(32ull * threadIdx.x), lcg_jump(32ull * MASK_THREADS),
              lcg_jump(32ull * MASK_THREADS * MASK_ILP - 32));
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags + (int64_t)r * max_steps + st), "r"(tag)
                 : "memory");
  }
}

void preload_mask_producer() {
  static const bool done = [] {
    cudaFuncAttributes at;
    return cudaFuncGetAttributes(&at, dropout_bits_step_kernel) == cudaSuccess;
  }();
  (void)done;
}

// ceil(keep * 2^53): keep-bit threshold on the 53-bit integer behind random()
static uint64_t keep_threshold(double keep) {
  if (!(keep > 0.0)) return 0;
  if (keep >= 1.0) return 1ull << 53;
  return (uint64_t)ceil(ldexp(keep, 53));
}

}  // namespace fs

using namespace fs;

extern "C" int fs_derive_seed_host(uint64_t master, const uint32_t* path, int32_t n_path,
                                   uint64_t* out) {
  if (!out || n_path < 0 || n_path > 8 || (n_path > 0 && !path)) {
    set_error("fs_derive_seed_host: invalid path");
    return FS_EINVAL;
  }
  *out = derive_seed(master, path, n_path);
  return FS_OK;
}

extern "C" int fs_train_seeds_host(uint64_t master, const int32_t* client_ids, const int32_t* cycles,
                                   int32_t n, uint64_t* out) {
  if (n < 0 || (n > 0 && (!client_ids || !cycles || !out))) {
    set_error("fs_train_seeds_host: invalid arguments");
    return FS_EINVAL;
  }
  for (int32_t i = 0; i < n; ++i)
    out[i] = derive_train_seed(master, (uint32_t)client_ids[i], (uint32_t)cycles[i]);
  return FS_OK;
}

extern "C" int fs_train_seeds(uint64_t master, const int32_t* client_ids, const int32_t* cycles,
                              int32_t n, uint64_t* seeds_out, void* stream) {
  if (n < 0) {
    set_error("fs_train_seeds: n < 0");
    return FS_EINVAL;
  }
  if (n == 0) return FS_OK;
  train_seeds_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(master, client_ids, cycles,
                                                                        n, seeds_out);
  return check_launch("train_seeds_kernel");
}

extern "C" int fs_shuffle_perms(const uint64_t* seeds, const int32_t* n_rows,
                                const int64_t* perm_off, int32_t n_req, int32_t epochs,
                                int32_t max_rows, int32_t* perm_out, void* stream) {
  if (n_req < 0 || epochs < 0 || max_rows < 0) {
    set_error("fs_shuffle_perms: invalid sizes");
    return FS_EINVAL;
  }
  if (n_req == 0 || epochs == 0) return FS_OK;
  if (max_rows <= 65536) {
    const size_t sm16 = SH_VB * sizeof(uint32_t) + (((size_t)max_rows * 2 + 15) & ~(size_t)15);
    if (sm16 > 48 * 1024) ensure_smem(shuffle16_kernel, (int)sm16);
    shuffle16_kernel<<<n_req * epochs, SH_THREADS, sm16, (cudaStream_t)stream>>>(seeds, n_rows, perm_off, epochs,
                                                                                 perm_out);
    return check_launch("shuffle16_kernel");
  }
  // larger shards: int32 chains staged in shared memory when they fit (swapping
  // in the output through L1/L2 with one-warp CTAs measured equal: latency-bound)
  const size_t smem = (size_t)max_rows * sizeof(int32_t);
  const int use_smem = smem <= 200 * 1024;
  if (use_smem && smem > 48 * 1024)
    ensure_smem(shuffle_kernel, (int)smem);
  shuffle_kernel<<<n_req * epochs, use_smem ? 128 : 32, use_smem ? smem : 0, (cudaStream_t)stream>>>(
      seeds, n_rows, perm_off, epochs, perm_out, use_smem);
  return check_launch("shuffle_kernel");
}

extern "C" int fs_dropout_bits(const uint64_t* seeds, const int32_t* n_rows, const int32_t* batch,
                               const int64_t* mask_off, int32_t n_req, int32_t epochs,
                               int32_t sum_hidden, double keep, uint32_t* bits_out, void* stream) {
  if (n_req < 0 || epochs < 0 || sum_hidden < 1) {
    set_error("fs_dropout_bits: invalid sizes");
    return FS_EINVAL;
  }
  if (n_req == 0 || epochs == 0) return FS_OK;
  const int64_t blocks = (int64_t)n_req * MASK_YSPLIT;
  dropout_bits_kernel<<<(unsigned)blocks, MASK_THREADS, 0, (cudaStream_t)stream>>>(
      seeds, n_rows, batch, mask_off, n_req, epochs, sum_hidden, keep_threshold(keep), bits_out);
  return check_launch("dropout_bits_kernel");
}

extern "C" int fs_dropout_bits_seed(uint64_t mask_seed, int64_t n_draws, double keep,
                                    uint32_t* bits_out, void* stream) {
  if (n_draws < 0) {
    set_error("fs_dropout_bits_seed: n_draws < 0");
    return FS_EINVAL;
  }
  if (n_draws == 0) return FS_OK;
  dropout_bits_seed_kernel<<<1, MASK_THREADS, 0, (cudaStream_t)stream>>>(mask_seed, n_draws,
                                                                         keep_threshold(keep), bits_out);
  return check_launch("dropout_bits_seed_kernel");
}

extern "C" int fs_dropout_bits_flagged(const uint64_t* seeds, const int32_t* n_rows, const int32_t* batch,
                                       const int64_t* mask_off, const int32_t* order, int32_t n_req, int32_t epochs,
                                       int32_t max_steps, int32_t sum_hidden, double keep, uint32_t* bits_out,
                                       int32_t* flags, int32_t tag, void* stream) {
  if (n_req < 0 || epochs < 0 || sum_hidden < 1 || max_steps < 0 || !flags || tag == 0) {
    set_error("fs_dropout_bits_flagged: invalid arguments");
    return FS_EINVAL;
  }
  if (n_req == 0 || epochs == 0 || max_steps == 0) return FS_OK;
  const int64_t blocks = (int64_t)n_req * max_steps;
  if (blocks > 0x7FFFFFFF) {
    set_error("fs_dropout_bits_flagged: too many (request, step) blocks");
    return FS_EINVAL;
  }
  dropout_bits_step_kernel<<<(unsigned)blocks, MASK_THREADS, 0, (cudaStream_t)stream>>>(
      seeds, n_rows, batch, mask_off, order, n_req, epochs, max_steps, sum_hidden, keep_threshold(keep), bits_out,
      flags, tag);
  return check_launch("dropout_bits_step_kernel");
}

