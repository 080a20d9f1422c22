// K5 (fp64 parity mode): batched per-client local SGD of the anomaly MLP.
//
// Replaces, for every client of a round at once:
//   client.train_local            pkg/src/fedsim/client.py:98-172
//   model.loss_and_grad/sgd_step  pkg/src/fedsim/model.py:189-221
//   backend loss_and_grad         pkg/src/fedsim/backends/_core.pyx:140-219
//   backend forward               pkg/src/fedsim/backends/_core.pyx:109-137
//
// Design (B200): one CTA owns one client for all of its steps (persistent
// grid, longest-first work queue), so the whole E x ceil(n/b) SGD chain of
// a client runs without a host round trip.  The client's parameters stay
// in its own HBM row (L2-resident while it trains: 418 KB for the
// 42-256-128-64-1 MLP), activations live in a per-CTA L2-resident scratch,
// and every layer product is a CTA-tiled fp64 tensor-core GEMM (64x64 tiles,
// 16-deep k chunks staged in shared memory, mma.sync m8n8k4 f64 per warp).  The SGD
// update p - lr*g is fused into the weight-gradient GEMM epilogue, written
// as an explicit (round(lr*g), then round(p - .)) pair so it matches the
// reference's `params.values - lr * grad.values` rounding.  Dropout
// keep-bits come from K3 (bit-exact numpy PCG64 streams); batch rows from
// K2's permutations.  The per-call loss_and_grad / forward entry points run
// the very same step code, which is what keeps
// train_local == fold(loss_and_grad + sgd_step) bitwise (tests/test_client).
#include <cstdio>

#include "fs_common.cuh"

namespace fs {
namespace f64 {

constexpr int THREADS = 512;
constexpr int TM = 64, TN = 64, TK = 32;
// warps tile the 64 x 64 CTA tile as WARPS_M x 4, each owning MB x 2 DMMA tiles
constexpr int WARPS_M = THREADS / 128, MB = 8 / WARPS_M, SLOTS = MB * 2 * 2;
static_assert(THREADS == 256 || THREADS == 512 || THREADS == 1024, "cta_gemm warp tiling");
constexpr int SPAD = 4;  // row padding: conflict-free DMMA fragment loads (rows k..k+3 x 8 columns)

struct GemmSmem {
  double As[TK][TM + SPAD];
  double Bs[TK][TN + SPAD];
  double Es[SLOTS][THREADS];  // per-thread epilogue operands, fetched by cp.async
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// fp64 tensor-core MMA, D[8x8] += A[8x4] . B[4x8]: lane (g = lane/4, t = lane%4)
// holds A[g][t], B[t][g] and D[g][2t], D[g][2t+1]. Each output's four products
// are added in k order with one rounding each, bit-identical to a chain of
// fma() over k (tests/test_gpu_dmma_probe.py).
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- operand views
struct RowMajor {  // (r, c) -> p[r*ld + c]
  const double* p;
  int64_t ld;
  __device__ __forceinline__ double operator()(int r, int c) const { return p[(int64_t)r * ld + c]; }
};
struct ColMajor {  // (r, c) -> p[c*ld + r]
  const double* p;
  int64_t ld;
  __device__ __forceinline__ double operator()(int r, int c) const { return p[(int64_t)c * ld + r]; }
};
struct GatherRows {  // batch rows of the shard: (m, k) -> X[rowidx[m]*d + k]
  const double* X;
  const int64_t* rowidx;
  int d;
  __device__ __forceinline__ double operator()(int m, int k) const { return X[rowidx[m] * d + k]; }
};
struct GatherRowsT {  // transposed: (m, k) -> X[rowidx[k]*d + m]
  const double* X;
  const int64_t* rowidx;
  int d;
  __device__ __forceinline__ double operator()(int m, int k) const { return X[rowidx[k] * d + m]; }
};

// C[M x N] = A[M x K] . B[K x N], handed element-wise to the epilogue. The k
// sum of every output runs sequentially 0..K-1, one rounding per product
// (fp64 DMMA over whole k4 slices, fma for a chunk's last K % 4), so a given
// shape always rounds identically, and like the reference's BLAS (shared by
// the batched and per-call paths).
//
// 64 x 64 CTA tile, 16-deep k chunks staged in shared memory (the next
// chunk's global loads are issued into registers before the current chunk's
// MMAs); the warps as WARPS_M x 4, each owning an 8MB x 16 block = MB x 2
// DMMA tiles.
//
// The epilogue is split in two: src(m, n) names the one double the output
// needs from memory (its bias, its previous W, its gating activation; nullptr
// for none), which the thread copies into its own shared-memory slots with
// cp.async when the tile starts, and fin(m, n, acc, e) combines and stores.
// The operand fetch so overlaps the tile's MMAs without holding registers;
// loaded inside fin instead, each of a thread's 16 outputs paid its own L2
// round trip (the stores may alias the loads as far as the compiler knows).
template <bool A_KCONTIG, bool B_NCONTIG, class LA, class LB, class SRC, class FIN>
__device__ void cta_gemm(int M, int N, int K, const LA& la, const LB& lb, const SRC& src,
                         const FIN& fin, GemmSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 2) * (8 * MB), wn = (warp & 3) * 16;
  // output slot s = (mb*2 + nb)*2 + c  ->  row wm + 8mb + g, column wn + 8nb + 2t + c
  auto out_m = [&](int s) { return wm + 8 * (s >> 2) + g; };
  auto out_n = [&](int s) { return wn + 8 * ((s >> 1) & 1) + 2 * t + (s & 1); };
  constexpr int QA = (TM * TK) / THREADS, QB = (TN * TK) / THREADS;
  auto a_pos = [&](int q, int& m, int& k) {
    const int idx = tid + q * THREADS;
    if (A_KCONTIG) {
      k = idx & (TK - 1);
      m = idx / TK;
    } else {
      m = idx & (TM - 1);
      k = idx / TM;
    }
  };
  auto b_pos = [&](int q, int& n, int& k) {
    const int idx = tid + q * THREADS;
    if (B_NCONTIG) {
      n = idx & (TN - 1);
      k = idx / TN;
    } else {
      k = idx & (TK - 1);
      n = idx / TK;
    }
  };
  for (int tm = 0; tm < M; tm += TM) {
    for (int tn = 0; tn < N; tn += TN) {
      double acc[SLOTS];
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        acc[s] = 0.0;
        const int m = tm + out_m(s), n = tn + out_n(s);
        const double* e = (m < M && n < N) ? src(m, n) : nullptr;
        if (e) cp_async8(&sm.Es[s][tid], e);
      }
      double ra[QA], rb[QB];
      auto fetch = [&](int k0) {
#pragma unroll
        for (int q = 0; q < QA; ++q) {
          int m, k;
          a_pos(q, m, k);
          const int gm = tm + m, gk = k0 + k;
          ra[q] = (gm < M && gk < K) ? la(gm, gk) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          int n, k;
          b_pos(q, n, k);
          const int gn = tn + n, gk = k0 + k;
          rb[q] = (gn < N && gk < K) ? lb(gk, gn) : 0.0;
        }
      };
      auto stage = [&]() {
#pragma unroll
        for (int q = 0; q < QA; ++q) {
          int m, k;
          a_pos(q, m, k);
          sm.As[k][m] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          int n, k;
          b_pos(q, n, k);
          sm.Bs[k][n] = rb[q];
        }
      };
      fetch(0);
      stage();
      __syncthreads();
      for (int k0 = 0; k0 < K; k0 += TK) {
        const bool more = k0 + TK < K;
        if (more) fetch(k0 + TK);
        const int kmax = min(TK, K - k0);
        const int k4 = kmax & ~3;
        for (int k = 0; k < k4; k += 4) {
          double a[MB], b[2];
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) a[mb] = sm.As[k + t][wm + 8 * mb + g];
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) b[nb] = sm.Bs[k + t][wn + 8 * nb + g];
#pragma unroll
          for (int mb = 0; mb < MB; ++mb)
#pragma unroll
            for (int nb = 0; nb < 2; ++nb) dmma_8x8x4(acc[(mb * 2 + nb) * 2], acc[(mb * 2 + nb) * 2 + 1], a[mb], b[nb]);
        }
        for (int k = k4; k < kmax; ++k) {  // the chunk's last K % 4 products
#pragma unroll
          for (int s = 0; s < SLOTS; ++s) acc[s] = fma(sm.As[k][out_m(s)], sm.Bs[k][out_n(s)], acc[s]);
        }
        __syncthreads();
        if (more) {
          stage();
          __syncthreads();
        }
      }
      cp_async_wait_all();
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        const int m = tm + out_m(s), n = tn + out_n(s);
        if (m < M && n < N) fin(m, n, acc[s], sm.Es[s][tid]);
      }
    }
  }
}

// ---------------------------------------------------------------- dropout masks
struct MaskView {
  int mode;              // FS_MASK_*
  double scale;          // value of a kept unit (bits mode)
  const uint32_t* bits;  // slot of this step
  const double* dense;   // layer-major [total_rows x h_l] blocks
  int total_rows;        // rows of the batch the masks were drawn for
  int row0;              // first row of this chunk inside that batch
  int base[FS_MAX_LAYERS];  // sum of hidden widths before hidden layer l
  // value multiplying relu(pre) of hidden layer `hl`, row m, unit n
  __device__ __forceinline__ double val(int hl, int m, int n, int width) const {
    const int64_t j = (int64_t)total_rows * base[hl] + (int64_t)(row0 + m) * width + n;
    if (mode == FS_MASK_BITS) return ((__ldg(bits + (j >> 5)) >> (j & 31)) & 1u) ? scale : 0.0;
    return __ldg(dense + j);
  }
};

__device__ __forceinline__ double sigmoid_one(double z) {  // _core.pyx:84-90
  if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
  const double e = exp(z);
  return e / (1.0 + e);
}

// numpy's pairwise summation of a float64 vector (np.sum; also what
// ndarray.sum(axis=0) does for a single column), as used by the reference
// for the head-bias gradient (_core.pyx:187) and width-1 bias gradients.
__device__ double np_pairwise_sum(const double* a, int n, int64_t stride) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += a[i * stride];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j * stride];
    int i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[(i + j) * stride];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i * stride];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2, stride) + np_pairwise_sum(a + n2 * stride, n - n2, stride);
}

// ---------------------------------------------------------------- one SGD step
struct StepBufs {
  double* H[FS_MAX_LAYERS + 1];  // H[l] for hidden outputs l=1..L-1 (scratch)
  double* D[2];                  // ping-pong activation gradients
};

enum StepMode { STEP_TRAIN = 0, STEP_GRAD = 1 };

// The parameter update of a training step: plain SGD p - lr*g written as the
// reference's two roundings (model.py:215-221), or the opt-in Adam with
// per-parameter moments m, v (same layout as W) and bias corrections
// c1 = 1 / (1 - b1^t), c2 = 1 / (1 - b2^t) of this step.
struct Opt {
  int adam;
  double b1, b2, eps, c1, c2;
  double *m, *v;
  __device__ __forceinline__ double apply(double w, int64_t i, double lr, double g) const {
    if (!adam) return __dsub_rn(w, __dmul_rn(lr, g));
    const double mi = b1 * m[i] + (1.0 - b1) * g;
    const double vi = b2 * v[i] + (1.0 - b2) * g * g;
    m[i] = mi;
    v[i] = vi;
    return w - lr * (mi * c1) / (sqrt(vi * c2) + eps);
  }
};

// Shared-memory per-step context (set up by the caller).
struct StepShared {
  int64_t* rowidx;  // [rows] absolute feature rows (nullptr-free: identity filled)
  double* y;        // [rows]
  double* z;        // [rows] logits (incl. bias)
  double* dz;       // [rows]
};

// One forward+backward(+update) of a batch of `rows` rows through the MLP.
// W: parameters (updated in place in STEP_TRAIN); G: gradient out (STEP_GRAD).
template <int MODE>
__device__ void mlp_step(const MlpLayout& lay, double* W, double* G, double lr, const double* X,
                         int rows, const StepShared& ss, const MaskView& mk, const StepBufs& bufs,
                         GemmSmem& sm, int* status, double* loss_out, const Opt& opt = Opt{}) {
  const int L = lay.L;
  const int tid = threadIdx.x;
  const int d0 = lay.f[0];

  // ---- forward through the hidden layers (relu, inverted dropout)
  for (int l = 0; l < L - 1; ++l) {
    const int K = lay.f[l], N = lay.f[l + 1];
    const double* Wl = W + lay.woff[l];
    const double* bl = W + lay.boff[l];
    double* Hout = bufs.H[l + 1];
    const int hl = l;
    auto src = [&](int, int n) { return bl + n; };
    auto fin = [&](int m, int n, double acc, double b) {
      double v = acc + b;
      v = v > 0.0 ? v : 0.0;
      if (mk.mode != FS_MASK_NONE) v = v * mk.val(hl, m, n, N);
      Hout[(int64_t)m * N + n] = v;
    };
    if (l == 0)
      cta_gemm<true, true>(rows, N, K, GatherRows{X, ss.rowidx, d0}, RowMajor{Wl, N}, src, fin, sm);
    else
      cta_gemm<true, true>(rows, N, K, RowMajor{bufs.H[l], K}, RowMajor{Wl, N}, src, fin, sm);
    __syncthreads();
  }

  // ---- head: logits, BCE gradient dz = (sigmoid(z) - y) / rows
  const int FL = lay.f[L - 1];
  const double* Hlast = (L - 1 >= 1) ? bufs.H[L - 1] : nullptr;
  const double* wh = W + lay.woff[L - 1];
  const double bh = W[lay.boff[L - 1]];
  {
    const int warp = tid >> 5, lane = tid & 31;
    for (int m = warp; m < rows; m += THREADS / 32) {
      double s = 0.0;
      for (int k = lane; k < FL; k += 32) {
        const double h = (L - 1 >= 1) ? Hlast[(int64_t)m * FL + k] : X[ss.rowidx[m] * d0 + k];
        s = fma(h, wh[k], s);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        const double z = s + bh;
        ss.z[m] = z;
        ss.dz[m] = (sigmoid_one(z) - ss.y[m]) / (double)rows;
        if (!isfinite(z)) atomicOr(status, 1);
      }
    }
  }
  __syncthreads();
  if (MODE == STEP_GRAD && tid == 0 && loss_out) {
    double loss = 0.0;
    for (int m = 0; m < rows; ++m) {
      const double z = ss.z[m];
      loss += (z > 0.0 ? z : 0.0) - z * ss.y[m] + log1p(exp(-fabs(z)));
    }
    *loss_out = loss / (double)rows;
  }

  // ---- head backward: D_{L-1} = gate(dz (x) w_head); then head update
  if (L >= 2) {
    double* Dn = bufs.D[(L - 1) & 1];
    const double* Hh = bufs.H[L - 1];
    const int hl = L - 2;
    for (int64_t e = tid; e < (int64_t)rows * FL; e += THREADS) {
      const int m = (int)(e / FL), k = (int)(e % FL);
      double v = ss.dz[m] * wh[k];
      const double h = Hh[e];
      if (h > 0.0) {
        if (mk.mode != FS_MASK_NONE) v = v * mk.val(hl, m, k, FL);
      } else {
        v = 0.0;
      }
      Dn[e] = v;
    }
  }
  __syncthreads();
  {
    double* wh_mut = W + lay.woff[L - 1];
    for (int k = tid; k < FL; k += THREADS) {
      double g = 0.0;
      for (int m = 0; m < rows; ++m) {
        const double h = (L >= 2) ? bufs.H[L - 1][(int64_t)m * FL + k] : X[ss.rowidx[m] * d0 + k];
        g = fma(h, ss.dz[m], g);
      }
      if (MODE == STEP_GRAD)
        G[lay.woff[L - 1] + k] = g;
      else
        wh_mut[k] = opt.apply(wh_mut[k], lay.woff[L - 1] + k, lr, g);
    }
    if (tid == THREADS - 1) {
      const double gb = np_pairwise_sum(ss.dz, rows, 1);
      if (MODE == STEP_GRAD)
        G[lay.boff[L - 1]] = gb;
      else
        W[lay.boff[L - 1]] = opt.apply(W[lay.boff[L - 1]], lay.boff[L - 1], lr, gb);
    }
  }
  __syncthreads();

  // ---- hidden layers, last to first
  for (int l = L - 2; l >= 0; --l) {
    const int K = lay.f[l], N = lay.f[l + 1];
    const double* Dn = bufs.D[(l + 1) & 1];  // gated grad wrt H_{l+1}  [rows x N]
    double* Wl = W + lay.woff[l];
    double* bl = W + lay.boff[l];
    if (l > 0) {  // D_l = gate(D_{l+1} . W_l^T, H_l)   (uses W_l before its update)
      double* Dl = bufs.D[l & 1];
      const double* Hl = bufs.H[l];
      const int hl = l - 1;
      auto src = [&](int m, int n) { return Hl + (int64_t)m * K + n; };
      auto fin = [&](int m, int n, double acc, double h) {
        double v = acc;
        if (h > 0.0) {
          if (mk.mode != FS_MASK_NONE) v = v * mk.val(hl, m, n, K);
        } else {
          v = 0.0;
        }
        Dl[(int64_t)m * K + n] = v;
      };
      cta_gemm<true, false>(rows, K, N, RowMajor{Dn, N}, ColMajor{Wl, N}, src, fin, sm);
      __syncthreads();
    }
    // G_l = H_l^T . D_{l+1}, fused with W_l -= lr * G_l
    if (MODE == STEP_GRAD) {
      double* Gl = G + lay.woff[l];
      auto src = [](int, int) -> const double* { return nullptr; };
      auto fin = [&](int m, int n, double acc, double) { Gl[(int64_t)m * N + n] = acc; };
      if (l == 0)
        cta_gemm<false, true>(K, N, rows, GatherRowsT{X, ss.rowidx, d0}, RowMajor{Dn, N}, src, fin, sm);
      else
        cta_gemm<false, true>(K, N, rows, ColMajor{bufs.H[l], K}, RowMajor{Dn, N}, src, fin, sm);
    } else {
      auto src = [&](int m, int n) -> const double* { return Wl + (int64_t)m * N + n; };
      auto fin = [&](int m, int n, double acc, double w) {
        const int64_t i = (int64_t)m * N + n;
        Wl[i] = opt.apply(w, lay.woff[l] + i, lr, acc);
      };
      if (l == 0)
        cta_gemm<false, true>(K, N, rows, GatherRowsT{X, ss.rowidx, d0}, RowMajor{Dn, N}, src, fin, sm);
      else
        cta_gemm<false, true>(K, N, rows, ColMajor{bufs.H[l], K}, RowMajor{Dn, N}, src, fin, sm);
    }
    // bias gradient: column sums of D_{l+1}, rows accumulated in order
    // (ndarray.sum(axis=0) adds rows in order, except that a single column
    // reduces pairwise like a 1-D sum)
    for (int n = tid; n < N; n += THREADS) {
      double gb;
      if (N == 1) {
        gb = np_pairwise_sum(Dn, rows, 1);
      } else {
        gb = Dn[n];
        for (int m = 1; m < rows; ++m) gb += Dn[(int64_t)m * N + n];
      }
      if (MODE == STEP_GRAD)
        G[lay.boff[l] + n] = gb;
      else
        bl[n] = opt.apply(bl[n], lay.boff[l] + n, lr, gb);
    }
    __syncthreads();
  }
}

// Forward only: probabilities of `rows` rows (eval or masked train mode).
__device__ void mlp_forward(const MlpLayout& lay, const double* W, const double* X, int rows,
                            const int64_t* rowidx, const MaskView& mk, const StepBufs& bufs,
                            GemmSmem& sm, double* probs) {
  const int L = lay.L;
  const int tid = threadIdx.x;
  const int d0 = lay.f[0];
  for (int l = 0; l < L - 1; ++l) {
    const int K = lay.f[l], N = lay.f[l + 1];
    const double* Wl = W + lay.woff[l];
    const double* bl = W + lay.boff[l];
    double* Hout = bufs.H[l + 1];
    const int hl = l;
    auto src = [&](int, int n) { return bl + n; };
    auto fin = [&](int m, int n, double acc, double b) {
      double v = acc + b;
      v = v > 0.0 ? v : 0.0;
      if (mk.mode != FS_MASK_NONE) v = v * mk.val(hl, m, n, N);
      Hout[(int64_t)m * N + n] = v;
    };
    if (l == 0)
      cta_gemm<true, true>(rows, N, K, GatherRows{X, rowidx, d0}, RowMajor{Wl, N}, src, fin, sm);
    else
      cta_gemm<true, true>(rows, N, K, RowMajor{bufs.H[l], K}, RowMajor{Wl, N}, src, fin, sm);
    __syncthreads();
  }
  const int FL = lay.f[L - 1];
  const double* wh = W + lay.woff[L - 1];
  const double bh = W[lay.boff[L - 1]];
  const int warp = tid >> 5, lane = tid & 31;
  for (int m = warp; m < rows; m += THREADS / 32) {
    double s = 0.0;
    for (int k = lane; k < FL; k += 32) {
      const double h = (L >= 2) ? bufs.H[L - 1][(int64_t)m * FL + k] : X[rowidx[m] * d0 + k];
      s = fma(h, wh[k], s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) probs[m] = sigmoid_one(s + bh);
  }
  __syncthreads();
}

// ---------------------------------------------------------------- kernels
struct TrainArgs {
  MlpLayout lay;
  fs_train_desc d;
  int64_t scratch_per_cta;  // doubles
  int* counter;
  double* scratch;
};

__device__ StepBufs carve(const MlpLayout& lay, double* base, int max_rows) {
  StepBufs b{};
  double* p = base;
  for (int l = 1; l < lay.L; ++l) {
    b.H[l] = p;
    p += (int64_t)max_rows * lay.f[l];
  }
  const int mh = lay.max_hidden > 0 ? lay.max_hidden : 1;
  b.D[0] = p;
  p += (int64_t)max_rows * mh;
  b.D[1] = p;
  return b;
}

__host__ __device__ inline int64_t scratch_doubles(const MlpLayout& lay, int max_rows) {
  int64_t s = 0;
  for (int l = 1; l < lay.L; ++l) s += (int64_t)max_rows * lay.f[l];
  const int mh = lay.max_hidden > 0 ? lay.max_hidden : 1;
  return s + 2 * (int64_t)max_rows * mh;
}

// Per-CTA global scratch of the batched trainer: the step buffers, then the
// batch's row indices, labels, logits and dz (L1/L2-resident; kept out of
// shared memory so TRAIN_CTAS_PER_SM CTAs fit on an SM at any max_batch).
constexpr int TRAIN_CTAS_PER_SM = 1;
__host__ __device__ inline int64_t train_scratch_doubles(const MlpLayout& lay, int max_rows) {
  return scratch_doubles(lay, max_rows) + 4 * (int64_t)max_rows;
}

__global__ void __launch_bounds__(THREADS, TRAIN_CTAS_PER_SM) train_kernel(TrainArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GemmSmem& sm = *reinterpret_cast<GemmSmem*>(smem_raw);
  const int maxb = a.d.max_batch;
  double* cta_scratch = a.scratch + (int64_t)blockIdx.x * a.scratch_per_cta;
  int64_t* rowidx = reinterpret_cast<int64_t*>(cta_scratch + scratch_doubles(a.lay, maxb));
  double* ysm = reinterpret_cast<double*>(rowidx + maxb);
  double* zsm = ysm + maxb;
  double* dzsm = zsm + maxb;
  __shared__ int s_item;

  const MlpLayout& lay = a.lay;
  const fs_train_desc& d = a.d;
  const StepBufs bufs = carve(lay, cta_scratch, maxb);
  const StepShared ss{rowidx, ysm, zsm, dzsm};

  while (true) {
    if (threadIdx.x == 0) s_item = atomicAdd(a.counter, 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= d.n_req) break;
    const int r = d.order[item];

    const int n = d.n_rows[r], B = d.batch[r];
    const int spe = (n + B - 1) / B;
    double* W = d.w_out + (int64_t)r * d.ldw;
    const double* W0 = reinterpret_cast<const double*>(d.w_start[r]);
    if (W0 != W)
      for (int64_t j = threadIdx.x; j < lay.M; j += THREADS) W[j] = W0[j];
    Opt opt{};
    if (d.optimizer == FS_OPT_ADAM) {  // moments start at zero for each request
      opt.adam = 1;
      opt.b1 = d.adam_beta1;
      opt.b2 = d.adam_beta2;
      opt.eps = d.adam_eps;
      opt.m = reinterpret_cast<double*>(d.opt_state) + (int64_t)r * 2 * d.ldw;
      opt.v = opt.m + d.ldw;
      for (int64_t j = threadIdx.x; j < lay.M; j += THREADS) opt.m[j] = opt.v[j] = 0.0;
    }
    __syncthreads();

    const int64_t slot_words = ((int64_t)B * lay.sum_hidden + 31) / 32;
    for (int step = d.start_step[r]; step < d.end_step[r]; ++step) {
      const int e = step / spe, s = step % spe;
      const int rows = min(B, n - s * B);
      const double lr = d.lr[(int64_t)r * d.epochs + e];
      const int32_t* perm_e = d.perm + d.perm_off[r] + (int64_t)e * n;
      for (int i = threadIdx.x; i < rows; i += THREADS) {
        const int64_t row = d.row_off[r] + perm_e[s * B + i];
        rowidx[i] = row;
        ysm[i] = d.labels[row];
      }
      MaskView mk{};
      mk.mode = d.mask_mode;
      mk.scale = d.scale;
      if (d.mask_mode == FS_MASK_BITS) mk.bits = d.mask_bits + d.mask_off[r] + (int64_t)step * slot_words;
      mk.total_rows = rows;
      mk.row0 = 0;
      int acc = 0;
      for (int l = 1; l < lay.L; ++l) {
        mk.base[l - 1] = acc;
        acc += lay.f[l];
      }
      __syncthreads();
      if (opt.adam) {
        opt.c1 = 1.0 / (1.0 - pow(opt.b1, (double)(step + 1)));
        opt.c2 = 1.0 / (1.0 - pow(opt.b2, (double)(step + 1)));
      }
      mlp_step<STEP_TRAIN>(lay, W, nullptr, lr, d.features, rows, ss, mk, bufs, sm,
                           d.status + r, nullptr, opt);
    }
    __syncthreads();
  }
}

struct GradArgs {
  MlpLayout lay;
  const double* W;
  const double* X;
  const double* Y;
  int rows;
  const double* dense;
  double* loss;
  double* grad;
  int* status;
  double* scratch;
};

__global__ void __launch_bounds__(THREADS) grad_kernel(GradArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GemmSmem& sm = *reinterpret_cast<GemmSmem*>(smem_raw);
  const int rows = a.rows;
  int64_t* rowidx = reinterpret_cast<int64_t*>(smem_raw + sizeof(GemmSmem));
  double* ysm = reinterpret_cast<double*>(rowidx + rows);
  double* zsm = ysm + rows;
  double* dzsm = zsm + rows;
  for (int i = threadIdx.x; i < rows; i += THREADS) {
    rowidx[i] = i;
    ysm[i] = a.Y[i];
  }
  const StepBufs bufs = carve(a.lay, a.scratch, rows);
  MaskView mk{};
  mk.mode = a.dense ? FS_MASK_DENSE : FS_MASK_NONE;
  mk.dense = a.dense;
  mk.total_rows = rows;
  int acc = 0;
  for (int l = 1; l < a.lay.L; ++l) {
    mk.base[l - 1] = acc;
    acc += a.lay.f[l];
  }
  __syncthreads();
  const StepShared ss{rowidx, ysm, zsm, dzsm};
  mlp_step<STEP_GRAD>(a.lay, const_cast<double*>(a.W), a.grad, 0.0, a.X, rows, ss, mk, bufs, sm,
                      a.status, a.loss);
}

constexpr int FWD_CHUNK = 128;

struct FwdArgs {
  MlpLayout lay;
  const double* W;
  const double* X;
  int rows;
  const double* dense;
  double* probs;
  double* scratch;
  int64_t scratch_per_cta;
};

__global__ void __launch_bounds__(THREADS) forward_kernel(FwdArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GemmSmem& sm = *reinterpret_cast<GemmSmem*>(smem_raw);
  int64_t* rowidx = reinterpret_cast<int64_t*>(smem_raw + sizeof(GemmSmem));
  const StepBufs bufs = carve(a.lay, a.scratch + (int64_t)blockIdx.x * a.scratch_per_cta, FWD_CHUNK);
  MaskView mk{};
  mk.mode = a.dense ? FS_MASK_DENSE : FS_MASK_NONE;
  mk.dense = a.dense;
  mk.total_rows = a.rows;
  int acc = 0;
  for (int l = 1; l < a.lay.L; ++l) {
    mk.base[l - 1] = acc;
    acc += a.lay.f[l];
  }
  for (int c0 = blockIdx.x * FWD_CHUNK; c0 < a.rows; c0 += gridDim.x * FWD_CHUNK) {
    const int rows = min(FWD_CHUNK, a.rows - c0);
    for (int i = threadIdx.x; i < rows; i += THREADS) rowidx[i] = c0 + i;
    mk.row0 = c0;
    __syncthreads();
    mlp_forward(a.lay, a.W, a.X, rows, rowidx, mk, bufs, sm, a.probs + c0);
  }
}

}  // namespace f64

// ============================================================== host entry points
using namespace f64;

static size_t train_smem_bytes(int max_batch) {
  return sizeof(GemmSmem) + (size_t)max_batch * (sizeof(int64_t) + 3 * sizeof(double));
}

static int train_grid(const fs_train_desc* d) {
  int g = d->grid > 0 ? d->grid : TRAIN_CTAS_PER_SM * kNumSMs;
  return g < d->n_req ? g : d->n_req;
}

}  // namespace fs

using namespace fs;

extern "C" size_t fs_train_workspace_bytes(const fs_train_desc* d) {
  MlpLayout lay;
  if (!d || make_layout(d->dims, d->n_dims, &lay) != FS_OK || d->n_req < 1) return 0;
  const int grid = train_grid(d);
  return 256 + (size_t)grid * train_scratch_doubles(lay, d->max_batch) * sizeof(double);
}

extern "C" int fs_train_f64(const fs_train_desc* d, void* stream) {
  MlpLayout lay;
  if (!d || make_layout(d->dims, d->n_dims, &lay) != FS_OK) {
    set_error("fs_train_f64: invalid layer dims");
    return FS_EINVAL;
  }
  if (d->n_req == 0) return FS_OK;
  if (d->n_req < 0 || d->max_batch < 1 || d->epochs < 0) {
    set_error("fs_train_f64: invalid sizes");
    return FS_EINVAL;
  }
  if (d->mask_mode != FS_MASK_NONE && d->mask_mode != FS_MASK_BITS) {
    set_error("fs_train_f64: mask_mode must be NONE or BITS");
    return FS_EINVAL;
  }
  if ((d->optimizer != FS_OPT_SGD && d->optimizer != FS_OPT_ADAM) ||
      (d->optimizer == FS_OPT_ADAM && (!d->opt_state || d->adam_eps <= 0.0))) {
    set_error("fs_train_f64: optimizer must be SGD, or ADAM with opt_state and eps > 0");
    return FS_EINVAL;
  }
  const size_t need = fs_train_workspace_bytes(d);
  if (d->workspace_bytes < need || !d->workspace) {
    set_error("fs_train_f64: workspace %zu < required %zu", d->workspace_bytes, need);
    return FS_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  TrainArgs a;
  a.lay = lay;
  a.d = *d;
  a.scratch_per_cta = train_scratch_doubles(lay, d->max_batch);
  a.counter = reinterpret_cast<int*>(d->workspace);
  a.scratch = reinterpret_cast<double*>(reinterpret_cast<char*>(d->workspace) + 256);
  if (cudaMemsetAsync(a.counter, 0, sizeof(int), st) != cudaSuccess) return check_launch("memset");
  const size_t smem = sizeof(GemmSmem);
  if (smem > 48 * 1024)
    ensure_smem(train_kernel, (int)smem);
  train_kernel<<<train_grid(d), THREADS, smem, st>>>(a);
  return check_launch("train_kernel");
}

extern "C" size_t fs_step_workspace_bytes(const int32_t* dims, int32_t n_dims, int32_t rows) {
  MlpLayout lay;
  if (make_layout(dims, n_dims, &lay) != FS_OK || rows < 1) return 0;
  return (size_t)scratch_doubles(lay, rows) * sizeof(double);
}

extern "C" int fs_loss_and_grad_f64(const int32_t* dims, int32_t n_dims, const double* w,
                                    const double* x, const double* y, int32_t rows,
                                    const double* dense_masks, double* loss_out, double* grad_out,
                                    int32_t* status, void* workspace, size_t workspace_bytes,
                                    void* stream) {
  MlpLayout lay;
  if (make_layout(dims, n_dims, &lay) != FS_OK || rows < 1) {
    set_error("fs_loss_and_grad_f64: invalid dims or rows");
    return FS_EINVAL;
  }
  if (workspace_bytes < fs_step_workspace_bytes(dims, n_dims, rows)) {
    set_error("fs_loss_and_grad_f64: workspace too small");
    return FS_EINVAL;
  }
  GradArgs a{lay, w, x, y, rows, dense_masks, loss_out, grad_out, status,
             reinterpret_cast<double*>(workspace)};
  const size_t smem = train_smem_bytes(rows);
  if (smem > 227 * 1024) {
    set_error("fs_loss_and_grad_f64: batch of %d rows exceeds shared-memory staging", rows);
    return FS_EINVAL;
  }
  if (smem > 48 * 1024)
    ensure_smem(grad_kernel, (int)smem);
  grad_kernel<<<1, THREADS, smem, (cudaStream_t)stream>>>(a);
  return check_launch("grad_kernel");
}

extern "C" size_t fs_forward_workspace_bytes(const int32_t* dims, int32_t n_dims, int32_t rows) {
  MlpLayout lay;
  if (make_layout(dims, n_dims, &lay) != FS_OK || rows < 1) return 0;
  int grid = (rows + FWD_CHUNK - 1) / FWD_CHUNK;
  if (grid > 4 * kNumSMs) grid = 4 * kNumSMs;
  return (size_t)grid * scratch_doubles(lay, FWD_CHUNK) * sizeof(double);
}

extern "C" int fs_forward_f64(const int32_t* dims, int32_t n_dims, const double* w, const double* x,
                              int32_t rows, const double* dense_masks, double* probs_out,
                              void* workspace, size_t workspace_bytes, void* stream) {
  MlpLayout lay;
  if (make_layout(dims, n_dims, &lay) != FS_OK || rows < 1) {
    set_error("fs_forward_f64: invalid dims or rows");
    return FS_EINVAL;
  }
  if (workspace_bytes < fs_forward_workspace_bytes(dims, n_dims, rows)) {
    set_error("fs_forward_f64: workspace too small");
    return FS_EINVAL;
  }
  int grid = (rows + FWD_CHUNK - 1) / FWD_CHUNK;
  if (grid > 4 * kNumSMs) grid = 4 * kNumSMs;
  FwdArgs a{lay, w, x, rows, dense_masks, probs_out, reinterpret_cast<double*>(workspace),
            scratch_doubles(lay, FWD_CHUNK)};
  const size_t smem = sizeof(GemmSmem) + FWD_CHUNK * sizeof(int64_t);
  if (smem > 48 * 1024)
    ensure_smem(forward_kernel, (int)smem);
  forward_kernel<<<grid, THREADS, smem, (cudaStream_t)stream>>>(a);
  return check_launch("forward_kernel");
}
