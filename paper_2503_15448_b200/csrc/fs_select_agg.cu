// K6 sign-alignment, K9 FedAvg sort keys, K7 FedAvg mean.
//
//   K6 fs_sign_align_f64   selection.calculate_relevance  selection.py:53-74
//                          backend sign_align_count        _core.pyx:222-236
//   K9 fs_gather_sort_keys server.aggregate's tobytes() sort key  server.py:84
//   K7 fs_aggregate_f64    server.aggregate's stacked mean   server.py:84-86
//
// Both K6 and K7 are HBM-streaming integer/float reductions: coalesced
// 16-byte loads, many independent loads in flight per thread, integer
// counts reduced with warp shuffles and one atomic per CTA.
#include "fs_common.cuh"
#include "fs_tc.cuh"

namespace fs {

constexpr int ALIGN_THREADS = 256;
constexpr int ALIGN_UNROLL = 4;                                    // double2 per thread per pass
constexpr int ALIGN_BLOCK_BYTES = 128 * 1024;  // client-row bytes streamed per CTA

template <class T>
__device__ __forceinline__ int sgn(T x) { return (x > T(0)) - (x < T(0)); }
// sign(a - b) for finite a, b: IEEE subtraction with gradual underflow is
// zero iff a == b and otherwise carries the ordering of a and b.
template <class T>
__device__ __forceinline__ int sgn_diff(T a, T b) { return (a > b) - (a < b); }

template <int MODE, class T>
__device__ __forceinline__ int aligned1(T c, T g, T p) {
  if (MODE == FS_ALIGN_WEIGHT_SIGN) return sgn(c) == sgn(g);
  return sgn_diff(c, g) == sgn_diff(g, p);
}

template <class T> struct Vec16;                       // 16-byte vector of T
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };

template <int MODE, class T>
__device__ __forceinline__ unsigned aligned_vec(const typename Vec16<T>::type& c, const typename Vec16<T>::type& g,
                                                const typename Vec16<T>::type& p) {
  const T* cc = reinterpret_cast<const T*>(&c);
  const T* gg = reinterpret_cast<const T*>(&g);
  const T* pp = reinterpret_cast<const T*>(&p);
  unsigned n = 0;
#pragma unroll
  for (int i = 0; i < Vec16<T>::n; ++i) n += aligned1<MODE, T>(cc[i], gg[i], pp[i]);
  return n;
}

template <int MODE, class T>
__global__ void __launch_bounds__(ALIGN_THREADS)
    sign_align_kernel(const uint64_t* wc, const uint64_t* wg, const uint64_t* wgp, int64_t M,
                      int blocks_per_req, unsigned long long* out) {
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
  const int r = blockIdx.x / blocks_per_req;
  const int blk = blockIdx.x % blocks_per_req;
  const T* c = reinterpret_cast<const T*>(wc[r]);
  const T* g = reinterpret_cast<const T*>(wg[r]);
  const T* p = MODE == FS_ALIGN_DELTA_SIGN ? reinterpret_cast<const T*>(wgp[r]) : nullptr;
  unsigned cnt = 0;
  const int64_t span = (M + blocks_per_req - 1) / blocks_per_req;
  const int64_t lo = (int64_t)blk * span;
  const int64_t hi = min(M, lo + span);
  const T zero = T(0);
  // 16-byte aligned bulk [v0, v1) of [lo, hi); scalar head/tail
  const uintptr_t mis = (reinterpret_cast<uintptr_t>(c + lo) | reinterpret_cast<uintptr_t>(g + lo) |
                         (p ? reinterpret_cast<uintptr_t>(p + lo) : 0)) & 15;
  const bool same_phase = ((reinterpret_cast<uintptr_t>(c) ^ reinterpret_cast<uintptr_t>(g)) & 15) == 0 &&
                          (!p || ((reinterpret_cast<uintptr_t>(c) ^ reinterpret_cast<uintptr_t>(p)) & 15) == 0);
  int64_t v0 = hi, v1 = hi;
  if (same_phase) {
    const int64_t head = mis ? (int64_t)((16 - (reinterpret_cast<uintptr_t>(c + lo) & 15)) / sizeof(T)) : 0;
    v0 = min(hi, lo + head);
    v1 = v0 + (hi - v0) / VN * VN;
  }
  for (int64_t j = lo + threadIdx.x; j < v0; j += ALIGN_THREADS)
    cnt += aligned1<MODE, T>(c[j], g[j], p ? p[j] : zero);
  const V* c2 = reinterpret_cast<const V*>(c + v0);
  const V* g2 = reinterpret_cast<const V*>(g + v0);
  const V* p2 = p ? reinterpret_cast<const V*>(p + v0) : nullptr;
  const int64_t nv = (v1 - v0) / VN;
  int64_t i = threadIdx.x;
  for (; i + (ALIGN_UNROLL - 1) * ALIGN_THREADS < nv; i += ALIGN_UNROLL * ALIGN_THREADS) {
    V cv[ALIGN_UNROLL], gv[ALIGN_UNROLL], pv[ALIGN_UNROLL];
#pragma unroll
    for (int u = 0; u < ALIGN_UNROLL; ++u) {
      cv[u] = __ldcs(c2 + i + u * ALIGN_THREADS);
      gv[u] = __ldg(g2 + i + u * ALIGN_THREADS);
      if (MODE == FS_ALIGN_DELTA_SIGN) pv[u] = __ldg(p2 + i + u * ALIGN_THREADS); else pv[u] = V{};
    }
#pragma unroll
    for (int u = 0; u < ALIGN_UNROLL; ++u) cnt += aligned_vec<MODE, T>(cv[u], gv[u], pv[u]);
  }
  for (; i < nv; i += ALIGN_THREADS) {
    const V pv = p2 ? p2[i] : V{};
    cnt += aligned_vec<MODE, T>(c2[i], g2[i], pv);
  }
  for (int64_t j = v1 + threadIdx.x; j < hi; j += ALIGN_THREADS)
    cnt += aligned1<MODE, T>(c[j], g[j], p ? p[j] : zero);
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  __shared__ unsigned warp_sums[ALIGN_THREADS / 32];
  if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned v = threadIdx.x < ALIGN_THREADS / 32 ? warp_sums[threadIdx.x] : 0u;
    v = __reduce_add_sync(0xffffffffu, v);
    if (threadIdx.x == 0 && v) atomicAdd(out + r, (unsigned long long)v);
  }
}

// Same count when every request compares against the SAME reference vectors
// (a synchronous round: all clients fetched one w_g / w_g_prev). A CTA takes
// one slice of the parameter range for G clients: the shared vectors are read
// once per slice and reused from registers, so HBM/L2 traffic is ~one stream
// per client row. Requires 16-byte aligned rows (rows are padded to 128 B).
template <int MODE, class T, int G>
__global__ void __launch_bounds__(ALIGN_THREADS)
    sign_align_shared_kernel(const uint64_t* wc, const T* __restrict__ g, const T* __restrict__ p, int n_req,
                             int64_t M, int blocks_per_grp, unsigned long long* out, uint64_t base = 0,
                             int64_t stride = 0) {
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
  const int grp = blockIdx.x / blocks_per_grp;
  const int blk = blockIdx.x % blocks_per_grp;
  const int r0 = grp * G;
  const int nq = min(G, n_req - r0);
  const T* c[G];
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int r = r0 + (q < nq ? q : 0);
    c[q] = reinterpret_cast<const T*>(wc ? wc[r] : base + (uint64_t)r * (uint64_t)stride);
  }
  const int64_t nvec = M / VN;
  const int64_t span = (nvec + blocks_per_grp - 1) / blocks_per_grp;
  const int64_t v0 = (int64_t)blk * span, v1 = min(nvec, v0 + span);
  unsigned cnt[G];
#pragma unroll
  for (int q = 0; q < G; ++q) cnt[q] = 0;
  const V* g2 = reinterpret_cast<const V*>(g);
  const V* p2 = reinterpret_cast<const V*>(p);
  for (int64_t i = v0 + threadIdx.x; i < v1; i += ALIGN_THREADS) {
    const V gv = __ldg(g2 + i);
    const V pv = MODE == FS_ALIGN_DELTA_SIGN ? __ldg(p2 + i) : V{};
    V cv[G];
#pragma unroll
    for (int q = 0; q < G; ++q)
      if (q < nq) cv[q] = __ldcs(reinterpret_cast<const V*>(c[q]) + i);
#pragma unroll
    for (int q = 0; q < G; ++q)
      if (q < nq) cnt[q] += aligned_vec<MODE, T>(cv[q], gv, pv);
  }
  if (blk == blocks_per_grp - 1) {  // scalar tail [nvec*VN, M)
    const T zero = T(0);
    for (int64_t j = nvec * VN + threadIdx.x; j < M; j += ALIGN_THREADS)
#pragma unroll
      for (int q = 0; q < G; ++q)
        if (q < nq) cnt[q] += aligned1<MODE, T>(c[q][j], g[j], MODE == FS_ALIGN_DELTA_SIGN ? p[j] : zero);
  }
  __shared__ unsigned warp_sums[G][ALIGN_THREADS / 32];
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const unsigned v = __reduce_add_sync(0xffffffffu, cnt[q]);
    if ((threadIdx.x & 31) == 0) warp_sums[q][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int q = 0; q < G; ++q) {
      unsigned v = threadIdx.x < ALIGN_THREADS / 32 ? warp_sums[q][threadIdx.x] : 0u;
      v = __reduce_add_sync(0xffffffffu, v);
      if (threadIdx.x == 0 && q < nq && v) atomicAdd(out + r0 + q, (unsigned long long)v);
    }
  }
}

__global__ void sort_keys_kernel(const uint64_t* rows, int k, int n_keys, uint64_t* keys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k * n_keys) return;
  const int row = i / n_keys, t = i % n_keys;
  const unsigned long long bits =
      (unsigned long long)__double_as_longlong(reinterpret_cast<const double*>(rows[row])[t]);
  keys[i] = __byte_perm((unsigned)(bits >> 32), 0, 0x0123) |
            ((uint64_t)__byte_perm((unsigned)bits, 0, 0x0123) << 32);
}

__global__ void sort_keys_f32_kernel(const uint64_t* rows, int k, int n_keys, uint64_t* keys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k * n_keys) return;
  const int row = i / n_keys, t = i % n_keys;
  const unsigned bits = __float_as_uint(reinterpret_cast<const float*>(rows[row])[t]);
  keys[i] = __byte_perm(bits, 0, 0x0123);
}

// ---------------------------------------------------------------- K9 on device
// Canonical order of k <= 1024 update rows by values.tobytes() without a host
// round trip: a bitonic sort in shared memory whose comparator looks at the
// leading 4 elements as big-endian integers (byte order of tobytes) and, on
// a tie, keeps scanning the rows element by element. Writes the row pointers
// in sorted order for the aggregation kernels.
constexpr int SORT_MAX = 1024;
constexpr int SORT_KEYS = 4;

template <class T>
__device__ __forceinline__ uint64_t be_key(T v);
template <>
__device__ __forceinline__ uint64_t be_key<double>(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return ((uint64_t)__byte_perm((unsigned)b, 0, 0x0123) << 32) | __byte_perm((unsigned)(b >> 32), 0, 0x0123);
}
template <>
__device__ __forceinline__ uint64_t be_key<float>(float v) {
  return __byte_perm(__float_as_uint(v), 0, 0x0123);
}

template <class T>
__device__ bool row_less(const uint64_t* keys, const uint64_t* rows, int a, int b, int nk, int64_t M) {
  for (int t = 0; t < nk; ++t) {
    const uint64_t ka = keys[a * SORT_KEYS + t], kb = keys[b * SORT_KEYS + t];
    if (ka != kb) return ka < kb;
  }
  const T* ra = reinterpret_cast<const T*>(rows[a]);
  const T* rb = reinterpret_cast<const T*>(rows[b]);
  for (int64_t j = nk; j < M; ++j) {
    const uint64_t ka = be_key<T>(ra[j]), kb = be_key<T>(rb[j]);
    if (ka != kb) return ka < kb;
  }
  return a < b;  // identical rows: any order gives the same sum
}

template <class T>
__global__ void __launch_bounds__(SORT_MAX) canonical_order_kernel(const uint64_t* rows, int k, int64_t M,
                                                                   uint64_t* sorted_rows,
                                                                   const int64_t* job_off = nullptr,
                                                                   const double* w_in = nullptr,
                                                                   double* w_sorted = nullptr) {
  if (job_off) {  // one CTA per aggregation job: rows[job_off[j], job_off[j+1])
    const int64_t o = job_off[blockIdx.x];
    rows += o;
    sorted_rows += o;
    if (w_in) {
      w_in += o;
      w_sorted += o;
    }
    k = (int)(job_off[blockIdx.x + 1] - o);
  }
  __shared__ uint64_t keys[SORT_MAX * SORT_KEYS];
  __shared__ int idx[SORT_MAX];
  const int nk = M < SORT_KEYS ? (int)M : SORT_KEYS;
  int n2 = 1;
  while (n2 < k) n2 <<= 1;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    idx[i] = i;
    if (i < k)
      for (int t = 0; t < nk; ++t) keys[i * SORT_KEYS + t] = be_key<T>(reinterpret_cast<const T*>(rows[i])[t]);
  }
  __syncthreads();
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const int a = idx[i], b = idx[j];
          const bool up = (i & size) == 0;
          // padding entries (>= k) sort last
          bool a_gt_b;
          if (a >= k)
            a_gt_b = (b < k) || (a > b);
          else if (b >= k)
            a_gt_b = false;
          else
            a_gt_b = row_less<T>(keys, rows, b, a, nk, M);
          if (a_gt_b == up) {
            idx[i] = b;
            idx[j] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    sorted_rows[i] = rows[idx[i]];
    if (w_in) w_sorted[i] = w_in[idx[i]];  // per-row weights follow their rows
  }
}

// ---------------------------------------------------------------- K7
// Ordered FedAvg column sums, out[j] = acc + rows[0][j] + rows[1][j] + ... in
// row order in float64, acc starting at -0.0 (-0.0 + x == x for every x):
// bitwise the reduction numpy's mean(axis=0) performs from the first row
// (server.py:84-86). The order is sequential per column, so parallelism is
// across columns only, and a thread's chain of loads must not stall on HBM
// latency: each CTA owns a 1 KB strip of every row and streams it with TMA
// bulk copies (cp.async.bulk, issued by warp 0, one lane per row) into a ring of AGG_STAGES x
// AGG_ROWS x 1 KB in shared memory (64 KB in flight per CTA, 3 CTAs per SM),
// completion tracked by mbarrier transaction counts; the 128 threads sum
// their 2 (float) or 1 (double) columns out of shared memory in row order.
// Rows whose pointers are not all 16-byte aligned, and a ragged last strip,
// take the scalar path (same order).
constexpr int AGG_THREADS = 128;
constexpr int AGG_STRIP = 1024;  // bytes of each row per CTA
constexpr int AGG_ROWS = 16;     // rows per stage
constexpr int AGG_STAGES = 4;
constexpr int AGG_RING = AGG_STAGES * AGG_ROWS * AGG_STRIP;

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tc::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
}

template <class T>
__device__ __forceinline__ double ordered_column_sum(const T* const* rows, int k, int64_t j,
                                                     const double* w = nullptr) {
  double acc = -0.0;
  if (w)  // product and sum rounded separately (no contraction): the oracle's restatement is exact
    for (int i = 0; i < k; ++i) acc = __dadd_rn(acc, __dmul_rn(w[i], (double)__ldcs(rows[i] + j)));
  else
    for (int i = 0; i < k; ++i) acc += (double)__ldcs(rows[i] + j);
  return acc;
}

// MEAN: out[j] = (ordered sum) / k as T (server.aggregate).
// !MEAN: out[j] = ordered sum as float64 (a rank's partial FedAvg sum; the
// ranks' sums are all-reduced and finished by mean_finish_kernel).
template <class T, bool MEAN, class OUT>
__global__ void __launch_bounds__(AGG_THREADS)
    ordered_rows_kernel(const uint64_t* rows, int k, int64_t M, OUT* out, const int64_t* job_off = nullptr,
                        const uint64_t* job_out = nullptr, const double* wts = nullptr) {
  if (job_off) {  // blockIdx.y = aggregation job: rows[job_off[j], job_off[j+1]) -> job_out[j]
    const int64_t o = job_off[blockIdx.y];
    rows += o;
    if (wts) wts += o;
    k = (int)(job_off[blockIdx.y + 1] - o);
    out = reinterpret_cast<OUT*>(job_out[blockIdx.y]);
  }
  constexpr int CPT = AGG_STRIP / (int)sizeof(T) / AGG_THREADS;  // columns per thread
  constexpr int64_t STRIP_COLS = AGG_STRIP / (int64_t)sizeof(T);
  extern __shared__ __align__(128) uint8_t agg_smem[];
  uint8_t* ring = agg_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(agg_smem + AGG_RING);
  const T** sh_rows = reinterpret_cast<const T**>(full + AGG_STAGES);
  double* sh_w = reinterpret_cast<double*>(sh_rows + k);  // weighted jobs: w[k], then their ordered sum
  const int tid = threadIdx.x;
  uint64_t mis = 0;
  for (int i = tid; i < k; i += AGG_THREADS) {
    sh_rows[i] = reinterpret_cast<const T*>(rows[i]);
    mis |= rows[i] & 15;
    if (wts) sh_w[i] = wts[i];
  }
  if (tid == 0) {
    for (int s = 0; s < AGG_STAGES; ++s) tc::mbar_init(&full[s], 1);
    tc::fence_mbar_init();
  }
  const bool vec_ok = !__syncthreads_or(mis != 0);
  double den = (double)k;
  if (wts) {  // weighted mean (staleness-weighted FedAvg, opt-in): sum w_i x_i / sum w_i, both in row order
    den = -0.0;
    for (int i = 0; i < k; ++i) den += sh_w[i];
  }
  const double* wrow = wts ? sh_w : nullptr;
  const int64_t col0 = (int64_t)blockIdx.x * STRIP_COLS;
  const int64_t ncols = min(STRIP_COLS, M - col0);
  auto emit = [&](int64_t j, double s) {
    if (MEAN) out[j] = (OUT)(s / den);
    else out[j] = (OUT)(s + 0.0);  // an all -0.0 column sums to +0.0
  };
  if (!vec_ok || ncols != STRIP_COLS) {
    for (int64_t c = tid; c < ncols; c += AGG_THREADS)
      emit(col0 + c, ordered_column_sum<T>(sh_rows, k, col0 + c, wrow));
    return;
  }
  const int nb = (k + AGG_ROWS - 1) / AGG_ROWS;
  // warp 0 refills a stage: lane 0 posts the byte count, lane r copies row r
  auto issue = [&](int b) {
    const int s = b % AGG_STAGES;
    const int nr = min(AGG_ROWS, k - b * AGG_ROWS);
    const int lane = tid & 31;
    if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)(nr * AGG_STRIP));
    __syncwarp();
    if (lane < nr)
      bulk_g2s(ring + (s * AGG_ROWS + lane) * AGG_STRIP, sh_rows[b * AGG_ROWS + lane] + col0, AGG_STRIP, &full[s]);
  };
  if (tid < 32)
    for (int b = 0; b < min(AGG_STAGES, nb); ++b) issue(b);
  {
    double acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = -0.0;
    for (int b = 0; b < nb; ++b) {
      const int s = b % AGG_STAGES;
      tc::mbar_wait(&full[s], (uint32_t)((b / AGG_STAGES) & 1));
      const int nr = min(AGG_ROWS, k - b * AGG_ROWS);
      const T* st = reinterpret_cast<const T*>(ring + s * AGG_ROWS * AGG_STRIP) + tid * CPT;
      if (wrow) {
        for (int r = 0; r < nr; ++r) {
          const T* e = st + r * STRIP_COLS;
          const double w = wrow[b * AGG_ROWS + r];
#pragma unroll
          for (int c = 0; c < CPT; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(w, (double)e[c]));
        }
      } else {
        for (int r = 0; r < nr; ++r) {
          const T* e = st + r * STRIP_COLS;
#pragma unroll
          for (int c = 0; c < CPT; ++c) acc[c] += (double)e[c];
        }
      }
      __syncthreads();  // stage s fully read
      if (tid < 32 && b + AGG_STAGES < nb) {
        tc::fence_async_smem();
        issue(b + AGG_STAGES);
      }
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) emit(col0 + tid * CPT + c, acc[c]);
  }
}

template <class T, bool MEAN, class OUT>
static int launch_ordered_rows(const uint64_t* rows, int k, int64_t M, OUT* out, cudaStream_t st, const char* what) {
  const size_t smem = AGG_RING + AGG_STAGES * sizeof(uint64_t) + (size_t)k * sizeof(void*);
  if (smem > 220 * 1024) {
    set_error("%s: k=%d updates exceed the staged pointer table", what, k);
    return FS_EINVAL;
  }
  auto kern = ordered_rows_kernel<T, MEAN, OUT>;
  ensure_smem(kern, (int)smem);
  const int64_t strips = (M * (int64_t)sizeof(T) + AGG_STRIP - 1) / AGG_STRIP;
  kern<<<(unsigned)strips, AGG_THREADS, smem, st>>>(rows, k, M, out, nullptr, nullptr, nullptr);
  return check_launch(what);
}

template <class T>
__global__ void mean_finish_kernel(const double* sum, double k, int64_t M, T* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < M) out[j] = (T)(sum[j] / k);
}

// M == 1: a single stacked column reduces pairwise (np.sum semantics).
__device__ double pairwise_rows(const uint64_t* rows, int lo, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += reinterpret_cast<const double*>(rows[lo + i])[0];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = reinterpret_cast<const double*>(rows[lo + j])[0];
    int i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += reinterpret_cast<const double*>(rows[lo + i + j])[0];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += reinterpret_cast<const double*>(rows[lo + i])[0];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_rows(rows, lo, n2) + pairwise_rows(rows, lo + n2, n - n2);
}

__global__ void aggregate_single_kernel(const uint64_t* rows, int k, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = pairwise_rows(rows, 0, k) / (double)k;
}

}  // namespace fs

using namespace fs;

template <class T>
static int sign_align_impl(const uint64_t* wc, const uint64_t* wg, const uint64_t* wg_prev, int32_t n_req,
                           int64_t M, int32_t mode, int64_t* aligned_out, void* stream) {
  if (n_req < 0 || M < 0 || (mode != FS_ALIGN_WEIGHT_SIGN && mode != FS_ALIGN_DELTA_SIGN) ||
      (mode == FS_ALIGN_DELTA_SIGN && !wg_prev)) {
    set_error("fs_sign_align_f64: invalid arguments");
    return FS_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (n_req == 0) return FS_OK;
  if (cudaMemsetAsync(aligned_out, 0, sizeof(int64_t) * n_req, st) != cudaSuccess)
    return check_launch("memset aligned");
  if (M == 0) return FS_OK;
  // ~128 KB of each client row per CTA (32 x 16-byte loads per thread): long
  // enough to amortise the CTA reduction, short enough for >= 2 waves
  const int64_t per_block = ALIGN_BLOCK_BYTES / (int64_t)sizeof(T);
  int bpr = (int)((M + per_block - 1) / per_block);
  // keep >= 2 waves of 8 resident CTAs per SM even for few requests
  const int64_t want = (int64_t)kNumSMs * 8 * 2;
  if ((int64_t)bpr * n_req < want) {
    const int64_t b2 = (want + n_req - 1) / n_req;
    const int64_t cap = (M + 255) / 256;
    bpr = (int)(b2 < cap ? b2 : cap);
    if (bpr < 1) bpr = 1;
  }
  const unsigned nblk = (unsigned)bpr * (unsigned)n_req;
  auto* out = reinterpret_cast<unsigned long long*>(aligned_out);
  if (mode == FS_ALIGN_WEIGHT_SIGN)
    sign_align_kernel<FS_ALIGN_WEIGHT_SIGN, T><<<nblk, ALIGN_THREADS, 0, st>>>(wc, wg, wg_prev, M, bpr, out);
  else
    sign_align_kernel<FS_ALIGN_DELTA_SIGN, T><<<nblk, ALIGN_THREADS, 0, st>>>(wc, wg, wg_prev, M, bpr, out);
  return check_launch("sign_align_kernel");
}

extern "C" int fs_sign_align_f64(const uint64_t* wc, const uint64_t* wg, const uint64_t* wg_prev,
                                 int32_t n_req, int64_t M, int32_t mode, int64_t* aligned_out, void* stream) {
  return sign_align_impl<double>(wc, wg, wg_prev, n_req, M, mode, aligned_out, stream);
}

extern "C" int fs_sign_align_f32(const uint64_t* wc, const uint64_t* wg, const uint64_t* wg_prev,
                                 int32_t n_req, int64_t M, int32_t mode, int64_t* aligned_out, void* stream) {
  return sign_align_impl<float>(wc, wg, wg_prev, n_req, M, mode, aligned_out, stream);
}

extern "C" int fs_gather_sort_keys_f64(const uint64_t* rows, int32_t k, int32_t n_keys,
                                       uint64_t* keys_out, void* stream) {
  if (k < 0 || n_keys < 0) {
    set_error("fs_gather_sort_keys_f64: invalid sizes");
    return FS_EINVAL;
  }
  const int total = k * n_keys;
  if (total == 0) return FS_OK;
  sort_keys_kernel<<<(total + 255) / 256, 256, 0, (cudaStream_t)stream>>>(rows, k, n_keys, keys_out);
  return check_launch("sort_keys_kernel");
}

extern "C" int fs_gather_sort_keys_f32(const uint64_t* rows, int32_t k, int32_t n_keys,
                                       uint64_t* keys_out, void* stream) {
  if (k < 0 || n_keys < 0) {
    set_error("fs_gather_sort_keys_f32: invalid sizes");
    return FS_EINVAL;
  }
  const int total = k * n_keys;
  if (total == 0) return FS_OK;
  sort_keys_f32_kernel<<<(total + 255) / 256, 256, 0, (cudaStream_t)stream>>>(rows, k, n_keys, keys_out);
  return check_launch("sort_keys_f32_kernel");
}

extern "C" int fs_aggregate_f32(const uint64_t* rows, int32_t k, int64_t M, float* out, void* stream) {
  if (k < 1 || M < 0) {
    set_error("fs_aggregate_f32: need k >= 1 updates");
    return FS_EINVAL;
  }
  if (M == 0) return FS_OK;
  return launch_ordered_rows<float, true, float>(rows, k, M, out, (cudaStream_t)stream, "fs_aggregate_f32");
}

extern "C" int fs_aggregate_f64(const uint64_t* rows, int32_t k, int64_t M, double* out,
                                void* stream) {
  if (k < 1 || M < 0) {
    set_error("fs_aggregate_f64: need k >= 1 updates");
    return FS_EINVAL;
  }
  if (M == 0) return FS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (M == 1) {
    aggregate_single_kernel<<<1, 32, 0, st>>>(rows, k, out);
    return check_launch("aggregate_single_kernel");
  }
  return launch_ordered_rows<double, true, double>(rows, k, M, out, st, "fs_aggregate_f64");
}

extern "C" int fs_sum_rows(const uint64_t* rows, int32_t k, int64_t M, int32_t dtype_bytes, double* out,
                           void* stream) {
  if (k < 0 || M < 0 || (dtype_bytes != 4 && dtype_bytes != 8)) {
    set_error("fs_sum_rows: invalid arguments");
    return FS_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (M == 0) return FS_OK;
  if (k == 0) {
    if (cudaMemsetAsync(out, 0, sizeof(double) * M, st) != cudaSuccess) return check_launch("memset sum");
    return FS_OK;
  }
  if (dtype_bytes == 8) return launch_ordered_rows<double, false, double>(rows, k, M, out, st, "fs_sum_rows");
  return launch_ordered_rows<float, false, double>(rows, k, M, out, st, "fs_sum_rows");
}

extern "C" int fs_mean_finish(const double* sum, int64_t k, int64_t M, int32_t dtype_bytes, void* out,
                              void* stream) {
  if (k < 1 || M < 0 || (dtype_bytes != 4 && dtype_bytes != 8)) {
    set_error("fs_mean_finish: invalid arguments");
    return FS_EINVAL;
  }
  if (M == 0) return FS_OK;
  const unsigned blocks = (unsigned)((M + 255) / 256);
  if (dtype_bytes == 8)
    mean_finish_kernel<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(sum, (double)k, M, (double*)out);
  else
    mean_finish_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(sum, (double)k, M, (float*)out);
  return check_launch("mean_finish_kernel");
}

// ---------------------------------------------------------------- client-sharded rounds, on the device
// One rank's share of a sharded synchronous round without a host round trip
// before the collective: its accepted rows (fs_select_rows job) are summed in
// canonical order into the exchange buffer's float64 head (fs_sum_job), its
// per-client counts / status / accepted count are scattered into the tail
// (fs_pack_exchange), the caller all-reduces the buffer (NCCL on the stream),
// and fs_mean_finish_dev writes sum / k -- or keeps the previous model when
// no rank accepted anything -- reading k from the reduced buffer.
extern "C" int fs_sum_job(const uint64_t* rows, const int64_t* job_off, int32_t max_k, int64_t M, int32_t dtype_bytes,
                          uint64_t* sorted_scratch, const uint64_t* job_out, void* stream) {
  if (max_k < 1 || max_k > SORT_MAX || M < 1 || (dtype_bytes != 4 && dtype_bytes != 8)) {
    set_error("fs_sum_job: need 1 <= max_k <= %d, M >= 1", SORT_MAX);
    return FS_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int threads = 32;
  while (threads < max_k && threads < SORT_MAX) threads <<= 1;
  const size_t smem = AGG_RING + AGG_STAGES * sizeof(uint64_t) + (size_t)max_k * (sizeof(void*) + sizeof(double));
  const int64_t strips = (M * (int64_t)dtype_bytes + AGG_STRIP - 1) / AGG_STRIP;
  if (dtype_bytes == 8) {
    canonical_order_kernel<double><<<1, threads, 0, st>>>(rows, 0, M, sorted_scratch, job_off);
    auto kern = ordered_rows_kernel<double, false, double>;
    ensure_smem(kern, (int)smem);
    kern<<<dim3((unsigned)strips, 1), AGG_THREADS, smem, st>>>(sorted_scratch, 0, M, nullptr, job_off, job_out,
                                                                nullptr);
  } else {
    canonical_order_kernel<float><<<1, threads, 0, st>>>(rows, 0, M, sorted_scratch, job_off);
    auto kern = ordered_rows_kernel<float, false, double>;
    ensure_smem(kern, (int)smem);
    kern<<<dim3((unsigned)strips, 1), AGG_THREADS, smem, st>>>(sorted_scratch, 0, M, nullptr, job_off, job_out,
                                                                nullptr);
  }
  return check_launch("fs_sum_job");
}

__global__ void pack_exchange_kernel(const int64_t* counts, const int32_t* status, const int32_t* own_idx, int k,
                                     int N, const int64_t* job_off, double* tail) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) {
    const int c = own_idx[i];
    tail[c] = counts ? (double)counts[i] : 0.0;
    tail[N + 1 + c] = (double)status[i];
  }
  if (i == 0) tail[N] = (double)job_off[1];
}

extern "C" int fs_pack_exchange(const int64_t* counts, const int32_t* status, const int32_t* own_idx, int32_t k,
                                int32_t N, const int64_t* job_off, double* tail, void* stream) {
  if (k < 0 || N < 1 || k > N || !status || !own_idx || !job_off || !tail) {
    set_error("fs_pack_exchange: invalid arguments");
    return FS_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(tail, 0, sizeof(double) * (2 * (size_t)N + 1), st) != cudaSuccess)
    return check_launch("memset exchange tail");
  pack_exchange_kernel<<<(unsigned)((k + 255) / 256 > 0 ? (k + 255) / 256 : 1), 256, 0, st>>>(counts, status, own_idx,
                                                                                          k, N, job_off, tail);
  return check_launch("pack_exchange_kernel");
}

template <class T>
__global__ void mean_finish_dev_kernel(const double* sum, const double* kp, int64_t M, const T* keep, T* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  const double k = *kp;
  out[j] = k > 0.0 ? (T)(sum[j] / k) : keep[j];
}

extern "C" int fs_mean_finish_dev(const double* sum, const double* k_dev, int64_t M, int32_t dtype_bytes,
                                  const void* keep, void* out, void* stream) {
  if (M < 1 || (dtype_bytes != 4 && dtype_bytes != 8) || !sum || !k_dev || !keep || !out) {
    set_error("fs_mean_finish_dev: invalid arguments");
    return FS_EINVAL;
  }
  const unsigned blocks = (unsigned)((M + 255) / 256);
  if (dtype_bytes == 8)
    mean_finish_dev_kernel<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(sum, k_dev, M, (const double*)keep,
                                                                             (double*)out);
  else
    mean_finish_dev_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(sum, k_dev, M, (const float*)keep,
                                                                            (float*)out);
  return check_launch("mean_finish_dev_kernel");
}

template <class T>
static int sign_align_shared_impl(const uint64_t* wc, const void* wg, const void* wgp, int32_t n_req, int64_t M,
                                  int32_t mode, int64_t* aligned_out, void* stream, uint64_t base = 0,
                                  int64_t stride = 0) {
  constexpr int G = 4;
  if (n_req < 0 || M < 0 || !wg || (mode != FS_ALIGN_WEIGHT_SIGN && mode != FS_ALIGN_DELTA_SIGN) ||
      (mode == FS_ALIGN_DELTA_SIGN && !wgp) || (reinterpret_cast<uintptr_t>(wg) & 15) ||
      (wgp && (reinterpret_cast<uintptr_t>(wgp) & 15))) {
    set_error("fs_sign_align_shared: invalid arguments (reference vectors must be 16-byte aligned)");
    return FS_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (n_req == 0) return FS_OK;
  if (cudaMemsetAsync(aligned_out, 0, sizeof(int64_t) * n_req, st) != cudaSuccess)
    return check_launch("memset aligned");
  if (M == 0) return FS_OK;
  const int groups = (n_req + G - 1) / G;
  // ~64 KB of each of the G client rows per CTA, >= 2 waves of 8 CTAs per SM
  int bpg = (int)((M * (int64_t)sizeof(T) + 65535) / 65536);
  const int64_t want = (int64_t)kNumSMs * 16;
  if ((int64_t)bpg * groups < want) bpg = (int)((want + groups - 1) / groups);
  const int64_t cap = (M + 1023) / 1024;
  if (bpg > cap) bpg = (int)(cap > 0 ? cap : 1);
  const unsigned nblk = (unsigned)bpg * (unsigned)groups;
  auto* out = reinterpret_cast<unsigned long long*>(aligned_out);
  const T* g = reinterpret_cast<const T*>(wg);
  const T* p = reinterpret_cast<const T*>(wgp);
  if (mode == FS_ALIGN_WEIGHT_SIGN)
    sign_align_shared_kernel<FS_ALIGN_WEIGHT_SIGN, T, G><<<nblk, ALIGN_THREADS, 0, st>>>(wc, g, p, n_req, M, bpg, out,
                                                                                     base, stride);
  else
    sign_align_shared_kernel<FS_ALIGN_DELTA_SIGN, T, G><<<nblk, ALIGN_THREADS, 0, st>>>(wc, g, p, n_req, M, bpg, out,
                                                                                    base, stride);
  return check_launch("sign_align_shared_kernel");
}

extern "C" int fs_sign_align_shared(const uint64_t* wc, const void* wg, const void* wg_prev, int32_t n_req,
                                    int64_t M, int32_t mode, int32_t dtype_bytes, int64_t* aligned_out,
                                    void* stream) {
  if (dtype_bytes == 8) return sign_align_shared_impl<double>(wc, wg, wg_prev, n_req, M, mode, aligned_out, stream);
  if (dtype_bytes == 4) return sign_align_shared_impl<float>(wc, wg, wg_prev, n_req, M, mode, aligned_out, stream);
  set_error("fs_sign_align_shared: dtype_bytes must be 4 or 8");
  return FS_EINVAL;
}

// Same count for rows at base + i * stride_bytes (a launch's output block):
// no pointer array, so a round needs no host-to-device copy for it.
extern "C" int fs_sign_align_rows(uint64_t base, int64_t stride_bytes, const void* wg, const void* wg_prev,
                                  int32_t n_req, int64_t M, int32_t mode, int32_t dtype_bytes, int64_t* aligned_out,
                                  void* stream) {
  if ((base & 15) || (stride_bytes & 15)) {
    set_error("fs_sign_align_rows: rows must be 16-byte aligned");
    return FS_EINVAL;
  }
  if (dtype_bytes == 8)
    return sign_align_shared_impl<double>(nullptr, wg, wg_prev, n_req, M, mode, aligned_out, stream, base, stride_bytes);
  if (dtype_bytes == 4)
    return sign_align_shared_impl<float>(nullptr, wg, wg_prev, n_req, M, mode, aligned_out, stream, base, stride_bytes);
  set_error("fs_sign_align_rows: dtype_bytes must be 4 or 8");
  return FS_EINVAL;
}

extern "C" int fs_canonical_order(const uint64_t* rows, int32_t k, int64_t M, int32_t dtype_bytes,
                                  uint64_t* sorted_rows, void* stream) {
  if (k < 0 || k > SORT_MAX || M < 1 || (dtype_bytes != 4 && dtype_bytes != 8)) {
    set_error("fs_canonical_order: need 0 <= k <= %d rows of M >= 1 elements", SORT_MAX);
    return FS_EINVAL;
  }
  if (k == 0) return FS_OK;
  int threads = 32;
  while (threads < k && threads < SORT_MAX) threads <<= 1;
  if (dtype_bytes == 8)
    canonical_order_kernel<double><<<1, threads, 0, (cudaStream_t)stream>>>(rows, k, M, sorted_rows);
  else
    canonical_order_kernel<float><<<1, threads, 0, (cudaStream_t)stream>>>(rows, k, M, sorted_rows);
  return check_launch("canonical_order_kernel");
}

// Many independent FedAvg means in one launch pair (the aggregations an
// asynchronous run queues between two training flushes): job j averages the
// rows rows[job_off[j] .. job_off[j+1]) in canonical byte order into
// job_out[j]. K9 orders every job's rows (one CTA per job) into
// sorted_scratch, then K7 runs with one grid row per job.
static int aggregate_jobs_impl(const uint64_t* rows, const double* weights, const int64_t* job_off, int32_t n_jobs,
                               int32_t max_k, int64_t M, int32_t dtype_bytes, uint64_t* sorted_scratch,
                               double* sorted_w, const uint64_t* job_out, void* stream) {
  if (n_jobs < 0 || max_k < 1 || max_k > SORT_MAX || M < 1 || (dtype_bytes != 4 && dtype_bytes != 8) ||
      n_jobs > 65535 || (weights && !sorted_w)) {
    set_error("fs_aggregate_jobs: need 0 <= n_jobs <= 65535 jobs of 1..%d rows, M >= 1", SORT_MAX);
    return FS_EINVAL;
  }
  if (n_jobs == 0) return FS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int threads = 32;
  while (threads < max_k && threads < SORT_MAX) threads <<= 1;
  const int esz = dtype_bytes;
  if (esz == 8)
    canonical_order_kernel<double><<<n_jobs, threads, 0, st>>>(rows, 0, M, sorted_scratch, job_off, weights, sorted_w);
  else
    canonical_order_kernel<float><<<n_jobs, threads, 0, st>>>(rows, 0, M, sorted_scratch, job_off, weights, sorted_w);
  int rc = check_launch("canonical_order_kernel (jobs)");
  if (rc != FS_OK) return rc;
  const size_t smem = AGG_RING + AGG_STAGES * sizeof(uint64_t) + (size_t)max_k * (sizeof(void*) + sizeof(double));
  const int64_t strips = (M * (int64_t)esz + AGG_STRIP - 1) / AGG_STRIP;
  const dim3 grid((unsigned)strips, (unsigned)n_jobs);
  const double* w = weights ? sorted_w : nullptr;
  if (esz == 8) {
    auto kern = ordered_rows_kernel<double, true, double>;
    ensure_smem(kern, (int)smem);
    kern<<<grid, AGG_THREADS, smem, st>>>(sorted_scratch, 0, M, nullptr, job_off, job_out, w);
  } else {
    auto kern = ordered_rows_kernel<float, true, float>;
    ensure_smem(kern, (int)smem);
    kern<<<grid, AGG_THREADS, smem, st>>>(sorted_scratch, 0, M, nullptr, job_off, job_out, w);
  }
  return check_launch("ordered_rows_kernel (jobs)");
}

// Many independent FedAvg means in one launch pair (the aggregations an
// asynchronous run queues between two training flushes): job j averages the
// rows rows[job_off[j] .. job_off[j+1]) in canonical byte order into
// job_out[j]. K9 orders every job's rows (one CTA per job) into
// sorted_scratch, then K7 runs with one grid row per job.
extern "C" int fs_aggregate_jobs(const uint64_t* rows, const int64_t* job_off, int32_t n_jobs, int32_t max_k,
                                 int64_t M, int32_t dtype_bytes, uint64_t* sorted_scratch, const uint64_t* job_out,
                                 void* stream) {
  return aggregate_jobs_impl(rows, nullptr, job_off, n_jobs, max_k, M, dtype_bytes, sorted_scratch, nullptr,
                             job_out, stream);
}

// Weighted variant (opt-in staleness-weighted FedAvg): job j's output is
// sum_i w_i x_i / sum_i w_i over its rows in canonical byte order (weights
// follow their rows through the ordering; float64 products and sums, each
// rounded, then the ordered weight sum). sorted_w holds job_off[n_jobs] doubles of scratch.
extern "C" int fs_aggregate_jobs_weighted(const uint64_t* rows, const double* weights, const int64_t* job_off,
                                          int32_t n_jobs, int32_t max_k, int64_t M, int32_t dtype_bytes,
                                          uint64_t* sorted_scratch, double* sorted_w, const uint64_t* job_out,
                                          void* stream) {
  if (!weights) {
    set_error("fs_aggregate_jobs_weighted: weights required");
    return FS_EINVAL;
  }
  return aggregate_jobs_impl(rows, weights, job_off, n_jobs, max_k, M, dtype_bytes, sorted_scratch, sorted_w,
                             job_out, stream);
}

// ---------------------------------------------------------------- K7, row-split (bf16 mode, one job)
// FedAvg of a synchronous round's accepted float32 rows when the numpy
// summation order is not the contract (bf16 mode is tolerance-matched): the
// k rows (canonical order, count read on the device from job_off[1]) are cut
// into SPLIT_G contiguous groups; CTA (strip, g) sums its group's rows over a
// 1024-column strip into float64 partials (4 columns per thread, 4 rows per
// load batch), and the finish pass adds the groups in order and divides by k.
// Deterministic for a given k; SPLIT_G x the column-strip parallelism of the
// sequential K7, which at the C4 row length has only 205 strips.
// Long rows (the WIDE model's 3.2M parameters) take 8 groups and 8-row load
// batches: 6.05 vs 5.20 TB/s at C5; the C4 row length keeps 16 x 4 (3.28 vs
// 2.64 TB/s for 8 x 8), measured with bench.hbm_microbench.
constexpr int SPLIT_THREADS = 256, SPLIT_COLS = 4 * SPLIT_THREADS;
constexpr int64_t SPLIT_LONG = 1 << 20;
inline int split_groups(int64_t M) { return M >= SPLIT_LONG ? 8 : 16; }

template <int SPLIT_G, int BATCH>
__global__ void __launch_bounds__(SPLIT_THREADS)
    rowsplit_partial_kernel(const uint64_t* rows, const int64_t* job_off, int64_t M, double* part) {
  const int k = (int)job_off[1];
  const int g = blockIdx.y;
  const int r0 = (int)((int64_t)k * g / SPLIT_G), r1 = (int)((int64_t)k * (g + 1) / SPLIT_G);
  const int64_t c = (int64_t)blockIdx.x * SPLIT_COLS + 4 * threadIdx.x;
  if (c >= M) return;
  double a0 = -0.0, a1 = -0.0, a2 = -0.0, a3 = -0.0;
  const bool vec = c + 4 <= M;
  int r = r0;
  if (vec) {
    for (; r + BATCH <= r1; r += BATCH) {
      float4 v[BATCH];
#pragma unroll
      for (int q = 0; q < BATCH; ++q)
        v[q] = __ldcs(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(rows[r + q]) + c));
#pragma unroll
      for (int q = 0; q < BATCH; ++q) {
        a0 += (double)v[q].x;
        a1 += (double)v[q].y;
        a2 += (double)v[q].z;
        a3 += (double)v[q].w;
      }
    }
  }
  for (; r < r1; ++r) {
    const float* row = reinterpret_cast<const float*>(rows[r]) + c;
    a0 += (double)row[0];
    if (c + 1 < M) a1 += (double)row[1];
    if (c + 2 < M) a2 += (double)row[2];
    if (c + 3 < M) a3 += (double)row[3];
  }
  double* p = part + (int64_t)g * M + c;
  p[0] = a0;
  if (c + 1 < M) p[1] = a1;
  if (c + 2 < M) p[2] = a2;
  if (c + 3 < M) p[3] = a3;
}

template <int SPLIT_G>
__global__ void rowsplit_finish_kernel(const double* part, const int64_t* job_off, int64_t M, const uint64_t* job_out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int k = (int)job_off[1];
  if (j >= M || k == 0) return;
  double s = -0.0;
#pragma unroll
  for (int g = 0; g < SPLIT_G; ++g) s += part[(int64_t)g * M + j];
  reinterpret_cast<float*>(job_out[0])[j] = (float)(s / (double)k);
}

extern "C" size_t fs_aggregate_rowsplit_workspace_bytes(int64_t M) {
  return M > 0 ? (size_t)split_groups(M) * (size_t)M * sizeof(double) : 0;
}

// One job (fs_select_rows output: rows in client order, job_off = {0, k},
// job_out[0]) of float32 rows, summed in that (deterministic) order: the
// canonical byte order only matters for numpy-bitwise parity, which is the
// fp64 mode's contract, so no K9 sort here. k = 0 writes nothing.
// sorted_scratch is unused (kept for the ABI).
extern "C" int fs_aggregate_rowsplit_f32(const uint64_t* rows, const int64_t* job_off, int32_t max_k, int64_t M,
                                         uint64_t* sorted_scratch, const uint64_t* job_out, void* workspace,
                                         size_t workspace_bytes, void* stream) {
  if (max_k < 1 || max_k > SORT_MAX || M < 1 || !workspace ||
      workspace_bytes < fs_aggregate_rowsplit_workspace_bytes(M)) {
    set_error("fs_aggregate_rowsplit_f32: invalid arguments or workspace");
    return FS_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  (void)sorted_scratch;
  double* part = reinterpret_cast<double*>(workspace);
  const unsigned strips = (unsigned)((M + SPLIT_COLS - 1) / SPLIT_COLS);
  if (split_groups(M) == 8) {
    rowsplit_partial_kernel<8, 8><<<dim3(strips, 8), SPLIT_THREADS, 0, st>>>(rows, job_off, M, part);
    if (int rc = check_launch("rowsplit_partial_kernel")) return rc;
    rowsplit_finish_kernel<8><<<(unsigned)((M + 255) / 256), 256, 0, st>>>(part, job_off, M, job_out);
  } else {
    rowsplit_partial_kernel<16, 4><<<dim3(strips, 16), SPLIT_THREADS, 0, st>>>(rows, job_off, M, part);
    if (int rc = check_launch("rowsplit_partial_kernel")) return rc;
    rowsplit_finish_kernel<16><<<(unsigned)((M + 255) / 256), 256, 0, st>>>(part, job_off, M, job_out);
  }
  return check_launch("rowsplit_finish_kernel");
}

// ---------------------------------------------------------------- selection on device
// filter_update (selection.py:77-85) for a synchronous round without a host
// round trip: accept[i] = aligned[i] / M >= theta (float64, inclusive), or
// every client when the round is unscored (delta_sign without movement
// history, server.py:283-284). The accepted rows (client order) become the
// single job of fs_aggregate_jobs: rows_out[0..k), job_off = {0, k},
// job_out[0] = out. One CTA, block-wide prefix sum.
__global__ void __launch_bounds__(1024) select_rows_kernel(const int64_t* aligned, int n, int64_t den, double theta,
                                                           int scored, int top_k, uint64_t base, int64_t stride,
                                                           uint64_t* rows_out, int64_t* job_off, uint64_t* job_out,
                                                           uint64_t out) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  extern __shared__ int64_t s_score[];  // [n] when top_k > 0
  if (threadIdx.x == 0) carry = 0;
  if (top_k > 0 && scored)
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_score[i] = aligned[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b0 = 0; b0 < n; b0 += blockDim.x) {
    const int i = b0 + threadIdx.x;
    int acc = i < n && (!scored || (double)aligned[i] / (double)den >= theta);
    if (acc && top_k > 0 && scored) {  // rank among all clients: higher score first, ties by index
      const int64_t si = s_score[i];
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const int64_t sj = s_score[j];
        rank += (sj > si) || (sj == si && j < i);
      }
      acc = rank < top_k;
    }
    const unsigned ball = __ballot_sync(0xffffffffu, acc);
    if (lane == 0) warp_tot[warp] = __popc(ball);
    __syncthreads();
    int before = carry;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    before += __popc(ball & ((1u << lane) - 1u));
    if (acc) rows_out[before] = base + (uint64_t)i * (uint64_t)stride;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += warp_tot[w];
      carry += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    job_off[0] = 0;
    job_off[1] = carry;
    job_out[0] = out;
  }
}

extern "C" int fs_select_rows(const int64_t* aligned, int32_t n, int64_t den, double theta, int32_t scored,
                              int32_t top_k, uint64_t base, int64_t stride_bytes, uint64_t* rows_out,
                              int64_t* job_off, uint64_t* job_out, uint64_t out, void* stream) {
  if (n < 0 || den < 1 || (scored && !aligned) || top_k < 0 || (top_k > 0 && n > 16384)) {
    set_error("fs_select_rows: invalid arguments");
    return FS_EINVAL;
  }
  const size_t smem = top_k > 0 && scored ? (size_t)n * sizeof(int64_t) : 0;
  if (smem > 48 * 1024) ensure_smem(select_rows_kernel, (int)smem);
  select_rows_kernel<<<1, 1024, smem, (cudaStream_t)stream>>>(aligned, n, den, theta, scored, top_k, base,
                                                              stride_bytes, rows_out, job_off, job_out, out);
  return check_launch("select_rows_kernel");
}

// ---------------------------------------------------------------- K6c: cosine relevance (opt-in)
// Opt-in `delta_cosine` selection (an extension: the reference counts
// matching signs, selection.py:53-74): score = cos(w_c - w_g, w_g - w_prev),
// the cosine between a client's update and the last global step, in float64
// with a fixed summation order (block b of row r reduces the columns
// [b*span, (b+1)*span) thread-strided, then a fixed xor-shuffle tree and warp
// order; the finish kernel adds the blocks in order), written as the
// fixed-point integer llrint(cos * 2^40) so the engines' integer score path
// (accept iff score / den >= theta, den = FS_COSINE_SCALE) carries it.
constexpr int COS_THREADS = 256, COS_BLOCKS = 32;

template <class T>
__global__ void __launch_bounds__(COS_THREADS)
    cosine_partial_kernel(const uint64_t* wc, uint64_t base, int64_t stride, const T* __restrict__ g,
                          const T* __restrict__ p, int64_t M, double* part) {
  const int r = blockIdx.y, b = blockIdx.x;
  const T* c = reinterpret_cast<const T*>(wc ? wc[r] : base + (uint64_t)r * (uint64_t)stride);
  const int64_t span = (M + gridDim.x - 1) / gridDim.x;
  const int64_t j0 = (int64_t)b * span, j1 = min(M, j0 + span);
  double d = 0.0, na = 0.0, nb = 0.0;
  for (int64_t j = j0 + threadIdx.x; j < j1; j += COS_THREADS) {
    const double gj = (double)g[j];
    const double a = (double)__ldcs(c + j) - gj, q = gj - (double)p[j];
    d = fma(a, q, d);
    na = fma(a, a, na);
    nb = fma(q, q, nb);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    d += __shfl_xor_sync(0xffffffffu, d, o);
    na += __shfl_xor_sync(0xffffffffu, na, o);
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
  }
  __shared__ double sh[COS_THREADS / 32][3];
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sh[warp][0] = d;
    sh[warp][1] = na;
    sh[warp][2] = nb;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < COS_THREADS / 32; ++w) t += sh[w][threadIdx.x];
    part[((int64_t)r * gridDim.x + b) * 3 + threadIdx.x] = t;
  }
}

__global__ void cosine_finish_kernel(const double* part, int n_req, int blocks, int64_t* score) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_req) return;
  double d = 0.0, na = 0.0, nb = 0.0;
  for (int b = 0; b < blocks; ++b) {
    d += part[((int64_t)r * blocks + b) * 3];
    na += part[((int64_t)r * blocks + b) * 3 + 1];
    nb += part[((int64_t)r * blocks + b) * 3 + 2];
  }
  const double cs = (na > 0.0 && nb > 0.0) ? fmin(1.0, fmax(-1.0, d / sqrt(na * nb))) : 0.0;
  score[r] = llrint(cs * (double)FS_COSINE_SCALE);
}

extern "C" size_t fs_cosine_align_workspace_bytes(int32_t n_req) {
  return n_req > 0 ? (size_t)n_req * COS_BLOCKS * 3 * sizeof(double) : 0;
}

extern "C" int fs_cosine_align(const uint64_t* wc, uint64_t base, int64_t stride_bytes, const void* wg,
                               const void* wg_prev, int32_t n_req, int64_t M, int32_t dtype_bytes, int64_t* score_out,
                               void* workspace, size_t workspace_bytes, void* stream) {
  if (n_req < 0 || M < 1 || !wg || !wg_prev || (dtype_bytes != 4 && dtype_bytes != 8) ||
      (!wc && (!base || stride_bytes <= 0))) {
    set_error("fs_cosine_align: invalid arguments");
    return FS_EINVAL;
  }
  if (n_req == 0) return FS_OK;
  if (!workspace || workspace_bytes < fs_cosine_align_workspace_bytes(n_req)) {
    set_error("fs_cosine_align: workspace %zu < required %zu", workspace_bytes, fs_cosine_align_workspace_bytes(n_req));
    return FS_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* part = reinterpret_cast<double*>(workspace);
  const dim3 grid(COS_BLOCKS, (unsigned)n_req);
  if (dtype_bytes == 8)
    cosine_partial_kernel<double><<<grid, COS_THREADS, 0, st>>>(wc, base, stride_bytes, (const double*)wg,
                                                                (const double*)wg_prev, M, part);
  else
    cosine_partial_kernel<float><<<grid, COS_THREADS, 0, st>>>(wc, base, stride_bytes, (const float*)wg,
                                                               (const float*)wg_prev, M, part);
  if (int rc = check_launch("cosine_partial_kernel")) return rc;
  cosine_finish_kernel<<<(n_req + 255) / 256, 256, 0, st>>>(part, n_req, COS_BLOCKS, score_out);
  return check_launch("cosine_finish_kernel");
}

