// K5 (bf16 mode) for MLPs whose hidden layers do not fit the on-chip
// trainers: the WIDE shape of BASELINE configs[4] (42-1024-1024-1024-1024-1).
// Same contract as fs_train_bf16 (client.train_local, client.py:98-172 with
// bf16 GEMM operands and fp32 masters): K2 permutations, K3 keep bits, per
// epoch learning rates, BCE on logits, plain SGD.
//
// A 1024x1024 layer (2 MB bf16, 4 MB fp32 master) cannot stay on one SM, so
// the clients of a launch train in lockstep instead: global SGD step t runs
// step t of every client that has one, each layer product being ONE batched
// GEMM over those clients (cublasGemmBatchedEx, bf16 x bf16 -> fp32; a plain
// library GEMM), with the elementwise work fused into small kernels between
// them:
//
//   forward   Z_{l+1} = H_l W_l            (GEMM)  ->  H_{l+1} = relu(Z + b) * keep * scale  (fwd_epilogue)
//   head      z = H_L w_h + b_h, dz = (sigmoid(z) - y) / rows, D_L = gate(dz w_h^T); head + b_{L-1} SGD (head_kernel)
//   backward  dH_l = D_{l+1} W_l^T          (GEMM)  ->  D_l = dH_l * gate(H_l); b_{l-1} SGD (gate_kernel)
//   update    W_l master += (-lr) H_l^T D_{l+1}   (GEMM with beta = 1: the SGD step IS the GEMM epilogue)
//   refresh   bf16 copies of the updated masters for the next step (convert_kernel)
//
// The fp32 masters live in the caller's output rows (w_out + r*ldw) from the
// first step on; workspace slots hold each client's bf16 weight copies and
// activations. Clients are processed in groups of at most WIDE_GROUP slots.
#include <cublas_v2.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "fs_common.cuh"

namespace fs {
namespace wide {

constexpr int WIDE_GROUP = 256;   // clients per lockstep group (workspace slots)
constexpr int MAXL = FS_MAX_LAYERS;

struct Geo {
  MlpLayout lay;
  int dp;                // input width padded to 16 (bf16 feature rows)
  int rb;                // activation rows per slot (max batch rounded up to 16)
  int64_t wb_off[MAXL];  // bf16 weight copy offsets (elements) inside a slot
  int64_t wb_elems;
  int64_t hid_base[MAXL];  // mask draw base of hidden layer l (1-based) within a step's block
  size_t slot_bytes;
  size_t x_off, h_off[MAXL], d_off[MAXL], t_off, y_off, z_off;  // byte offsets inside a slot
};

// head-logit partials per row: one per warp of the last forward epilogue's
// grid (256-thread blocks over the last hidden width), summed in a fixed order
// by the consumer so the logits do not depend on atomic arrival order
__host__ __device__ __forceinline__ int zparts(int n_last) { return (n_last + 255) / 256 * 8; }

static bool make(const fs_train_desc* d, Geo* g) {
  if (make_layout(d->dims, d->n_dims, &g->lay) != FS_OK) return false;
  const MlpLayout& L = g->lay;
  if (L.L < 2 || L.L > MAXL) return false;
  g->dp = (L.f[0] + 15) / 16 * 16;
  g->rb = std::max(16, (d->max_batch + 15) / 16 * 16);
  int64_t o = 0;
  for (int l = 0; l < L.L - 1; ++l) {  // hidden weight matrices; the head stays fp32
    g->wb_off[l] = o;
    o += (int64_t)(l == 0 ? g->dp : L.f[l]) * L.f[l + 1];
  }
  g->wb_elems = o;
  int64_t hb = 0;
  for (int l = 1; l < L.L; ++l) {
    g->hid_base[l] = hb;
    hb += L.f[l];
  }
  size_t s = (size_t)g->wb_elems * 2;
  auto take = [&](size_t bytes) {
    s = (s + 255) / 256 * 256;
    const size_t at = s;
    s += bytes;
    return at;
  };
  g->x_off = take((size_t)g->rb * g->dp * 2);
  for (int l = 1; l < L.L; ++l) {
    g->h_off[l] = take((size_t)g->rb * L.f[l] * 2);
    g->d_off[l] = take((size_t)g->rb * L.f[l] * 2);
  }
  g->t_off = take((size_t)g->rb * L.max_hidden * 4);
  g->y_off = take((size_t)g->rb * 4 * 2);  // labels, dz
  g->z_off = take((size_t)g->rb * zparts(L.f[L.L - 1]) * 4);  // head-logit partials (last forward epilogue)
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
};

// ------------------------------------------------------------------ kernels
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
  int dp;
  int64_t wb_off[MAXL];
  size_t slot_bytes;
  uint8_t* slots;
  float* w_out;
  int64_t ldw;
};

// bf16 copies of every hidden weight matrix of the listed clients (W_0 rows
// padded to dp with zeros, matching the zero-padded feature columns): one
// 16-byte read and one 8-byte write per 4 parameters (fout % 4 == 0).
__global__ void convert_kernel(ConvArgs c, const StepRow* rows, int n) {
  const int a = blockIdx.y;
  if (a >= n) return;
  const StepRow sr = rows[a];
  const float* m = c.w_out + (int64_t)sr.req * c.ldw;
  __nv_bfloat16* wb = reinterpret_cast<__nv_bfloat16*>(c.slots + (size_t)sr.slot * c.slot_bytes);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int l = 0; l < c.lay.L - 1; ++l) {
    const int fin = c.lay.f[l], fout = c.lay.f[l + 1];
    const float* src = m + c.lay.woff[l];
    __nv_bfloat16* dst = wb + c.wb_off[l];
    const int64_t real = (int64_t)fin * fout;
    const int64_t total = (int64_t)(l == 0 ? c.dp : fin) * fout;
    const bool vec = (fout % 4 == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(dst) & 7) == 0);
    if (vec) {
      for (int64_t j4 = t0; j4 < total / 4; j4 += stride) {
        const int64_t j = j4 * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < real) v = __ldcs(reinterpret_cast<const float4*>(src + j));
        __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 packed;
        packed.x = *reinterpret_cast<uint32_t*>(&lo);
        packed.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(dst + j) = packed;
      }
    } else {
      for (int64_t j = t0; j < total; j += stride) dst[j] = __float2bfloat16_rn(j < real ? src[j] : 0.f);
    }
  }
}

struct StepArgs {
  MlpLayout lay;
  int dp, rb;
  int64_t hid_base[MAXL];
  size_t slot_bytes, x_off, h_off[MAXL], d_off[MAXL], t_off, y_off, z_off;
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
};

__device__ __forceinline__ uint8_t* slot_of(const StepArgs& a, int slot) { return a.slots + (size_t)slot * a.slot_bytes; }

// X rows of the step (permuted shard rows, bf16, zero padded) and labels
__global__ void gather_kernel(StepArgs a, const StepRow* rows) {
  const StepRow sr = rows[blockIdx.x];
  uint8_t* sb = slot_of(a, sr.slot);
  __nv_bfloat16* x = reinterpret_cast<__nv_bfloat16*>(sb + a.x_off);
  float* y = reinterpret_cast<float*>(sb + a.y_off);
  const int n = a.n_rows[sr.req], B = a.batch[sr.req];
  const int32_t* perm = a.perm + a.perm_off[sr.req] + (int64_t)sr.e * n + (int64_t)sr.s * B;
  const int64_t base = a.row_off[sr.req];
  const int cpr = a.dp / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < a.rb * cpr; i += blockDim.x) {
    const int r = i / cpr, c = i % cpr;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < sr.rows) v = *reinterpret_cast<const uint4*>(a.feat + (base + perm[r]) * a.dp + c * 8);
    *reinterpret_cast<uint4*>(x + (int64_t)r * a.dp + c * 8) = v;
  }
  for (int r = threadIdx.x; r < a.rb; r += blockDim.x) y[r] = r < sr.rows ? a.labels[base + perm[r]] : 0.f;
}

__device__ __forceinline__ bool keep_bit(const StepArgs& a, const StepRow& sr, int l, int r, int u) {
  if (a.mask_mode != FS_MASK_BITS) return true;
  const int B = a.batch[sr.req];
  const int64_t slot_words = ((int64_t)B * a.lay.sum_hidden + 31) / 32;
  const uint32_t* bits = a.mask_bits + a.mask_off[sr.req] + (int64_t)sr.global_step * slot_words;
  const int64_t j = (int64_t)sr.rows * a.hid_base[l] + (int64_t)r * a.lay.f[l] + u;
  return (bits[j >> 5] >> (j & 31)) & 1u;
}

// H_l = relu(Z + b_{l-1}) * keep * scale  (bf16), Z in the fp32 temp. The
// last hidden layer also forms the head logits from the fp32 values (as the
// on-chip trainers do): per-warp partials of sum_u H[r][u] w_h[u].
__global__ void fwd_epilogue_kernel(StepArgs a, const StepRow* rows, int l) {
  const StepRow sr = rows[blockIdx.y];
  const int N = a.lay.f[l];
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const bool last = l == a.lay.L - 1;
  uint8_t* sb = slot_of(a, sr.slot);
  const float* z = reinterpret_cast<const float*>(sb + a.t_off);
  __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(sb + a.h_off[l]);
  float* zacc = reinterpret_cast<float*>(sb + a.z_off);
  const float* W = a.w_out + (int64_t)sr.req * a.ldw;
  const float b = u < N ? W[a.lay.boff[l - 1] + u] : 0.f;
  const float wh = last && u < N ? W[a.lay.woff[l] + u] : 0.f;
  const float sc = a.mask_mode == FS_MASK_BITS ? a.scale : 1.f;
  for (int r = 0; r < a.rb; ++r) {
    float v = 0.f;
    if (r < sr.rows && u < N) {
      v = fmaxf(z[(int64_t)r * N + u] + b, 0.f);
      v = keep_bit(a, sr, l, r, u) ? v * sc : 0.f;
    }
    if (u < N) h[(int64_t)r * N + u] = __float2bfloat16_rn(v);
    if (last && r < sr.rows) {
      float p = v * wh;
      for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
      if ((threadIdx.x & 31) == 0) zacc[(int64_t)r * zparts(N) + blockIdx.x * 8 + (threadIdx.x >> 5)] = p;
    }
  }
}

// head: logits, dz, D_{L-1}, SGD on the head and on b_{L-2}; one CTA per client
__global__ void __launch_bounds__(256) head_kernel(StepArgs a, const StepRow* rows) {
  const StepRow sr = rows[blockIdx.x];
  const int L = a.lay.L, N = a.lay.f[L - 1];
  uint8_t* sb = slot_of(a, sr.slot);
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(sb + a.h_off[L - 1]);
  __nv_bfloat16* dout = reinterpret_cast<__nv_bfloat16*>(sb + a.d_off[L - 1]);
  const float* y = reinterpret_cast<const float*>(sb + a.y_off);
  float* dz = reinterpret_cast<float*>(sb + a.y_off) + a.rb;
  float* W = a.w_out + (int64_t)sr.req * a.ldw;
  float* wh = W + a.lay.woff[L - 1];
  float* bh = W + a.lay.boff[L - 1];
  float* bprev = W + a.lay.boff[L - 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ float s_dz[1024];
  __shared__ float s_red[8];
  const float* zacc = reinterpret_cast<const float*>(sb + a.z_off);
  for (int r = threadIdx.x; r < a.rb; r += blockDim.x) {
    float d = 0.f;
    if (r < sr.rows) {
      const int zp = zparts(N);
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
  for (int u = threadIdx.x; u < N; u += blockDim.x) {
    const float w = wh[u];
    float g = 0.f, gb = 0.f;
    for (int r = 0; r < a.rb; ++r) {
      const float hv = __bfloat162float(h[(int64_t)r * N + u]);
      g = fmaf(hv, s_dz[r], g);
      const __nv_bfloat16 dv = __float2bfloat16_rn(hv > 0.f ? s_dz[r] * w * sc : 0.f);
      dout[(int64_t)r * N + u] = dv;
      gb += __bfloat162float(dv);
    }
    wh[u] = w - sr.lr * g;
    bprev[u] -= sr.lr * gb;
  }
  float t = 0.f;
  for (int r = threadIdx.x; r < a.rb; r += blockDim.x) t += s_dz[r];
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) s_red[warp] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w2 = 0; w2 < 8; ++w2) s += s_red[w2];
    bh[0] -= sr.lr * s;
  }
}

// D_l = dH_l * scale * [H_l > 0] (bf16) and SGD on b_{l-1}
__global__ void gate_kernel(StepArgs a, const StepRow* rows, int l) {
  const StepRow sr = rows[blockIdx.y];
  const int N = a.lay.f[l];
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= N) return;
  uint8_t* sb = slot_of(a, sr.slot);
  const float* dh = reinterpret_cast<const float*>(sb + a.t_off);
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(sb + a.h_off[l]);
  __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(sb + a.d_off[l]);
  const float sc = a.mask_mode == FS_MASK_BITS ? a.scale : 1.f;
  float gb = 0.f;
  for (int r = 0; r < a.rb; ++r) {
    const float hv = __bfloat162float(h[(int64_t)r * N + u]);
    const __nv_bfloat16 dv = __float2bfloat16_rn(hv > 0.f ? dh[(int64_t)r * N + u] * sc : 0.f);
    d[(int64_t)r * N + u] = dv;
    gb += __bfloat162float(dv);
  }
  a.w_out[(int64_t)sr.req * a.ldw + a.lay.boff[l - 1] + u] -= sr.lr * gb;
}

// ------------------------------------------------------------------ host
static cublasHandle_t blas() {
  static std::mutex mu;
  static std::map<int, cublasHandle_t> per_device;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = per_device.find(dev);
  if (it != per_device.end()) return it->second;
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
  per_device[dev] = h;
  return h;
}

static int blas_ok(cublasStatus_t s, const char* what) {
  if (s == CUBLAS_STATUS_SUCCESS) return FS_OK;
  set_error("fs_train_bf16 (wide): %s failed (cuBLAS status %d)", what, (int)s);
  return FS_ECUDA;
}

}  // namespace wide

size_t wide_workspace_bytes(const fs_train_desc* d) {
  wide::Geo g;
  if (!d || d->n_req < 1 || !wide::make(d, &g)) return 0;
  const size_t G = (size_t)std::min(d->n_req, wide::WIDE_GROUP);
  // slots + per-step staging (rows + pointer arrays)
  return G * g.slot_bytes + 256 + G * (sizeof(wide::StepRow) + 3 * 8 * (size_t)(3 * FS_MAX_LAYERS)) + 65536;
}

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
  cublasHandle_t h = blas();
  if (!h) {
    set_error("fs_train_bf16 (wide): cublasCreate failed");
    return FS_ECUDA;
  }
  if (int rc = blas_ok(cublasSetStream(h, st), "cublasSetStream")) return rc;
  // per-request geometry on the host (the descriptor's arrays live in HBM)
  std::vector<int32_t> nr(n), bt(n), s0(n), s1(n);
  std::vector<double> lr((size_t)n * std::max(d->epochs, 1));
  cudaMemcpyAsync(nr.data(), d->n_rows, 4 * (size_t)n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(bt.data(), d->batch, 4 * (size_t)n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(s0.data(), d->start_step, 4 * (size_t)n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(s1.data(), d->end_step, 4 * (size_t)n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(lr.data(), d->lr, 8 * lr.size(), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("wide: metadata");
  for (int r = 0; r < n; ++r)
    if (bt[r] > g.rb || bt[r] < 1) {
      set_error("fs_train_bf16 (wide): batch %d exceeds max_batch", bt[r]);
      return FS_EINVAL;
    }

  const size_t G = (size_t)std::min(n, WIDE_GROUP);
  uint8_t* ws = reinterpret_cast<uint8_t*>(d->workspace);
  uint8_t* slots = ws;
  uint8_t* stage = ws + G * g.slot_bytes;  // device staging: StepRow[] then pointer arrays
  float* w_out = reinterpret_cast<float*>(d->w_out);

  StepArgs sa;
  sa.lay = L;
  sa.dp = g.dp;
  sa.rb = g.rb;
  for (int l = 0; l < MAXL; ++l) {
    sa.hid_base[l] = g.hid_base[l];
    sa.h_off[l] = g.h_off[l];
    sa.d_off[l] = g.d_off[l];
  }
  sa.slot_bytes = g.slot_bytes;
  sa.x_off = g.x_off;
  sa.t_off = g.t_off;
  sa.y_off = g.y_off;
  sa.z_off = g.z_off;
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
  ConvArgs ca;
  ca.lay = L;
  ca.dp = g.dp;
  for (int l = 0; l < MAXL; ++l) ca.wb_off[l] = g.wb_off[l];
  ca.slot_bytes = g.slot_bytes;
  ca.slots = slots;
  ca.w_out = w_out;
  ca.ldw = d->ldw;

  const float one = 1.f, zero = 0.f;
  const int H = L.L - 1;  // hidden layers
  for (int g0 = 0; g0 < n; g0 += (int)G) {
    const int gn = std::min((int)G, n - g0);
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
      const size_t rb = (sizeof(StepRow) * gn + 255) / 256 * 256;
      std::vector<uint8_t> host(rb + 4 * (size_t)gn);
      memcpy(host.data(), all.data(), sizeof(StepRow) * gn);
      memcpy(host.data() + rb, reqs.data(), 4 * (size_t)gn);
      cudaMemcpyAsync(stage, host.data(), host.size(), cudaMemcpyHostToDevice, st);
      dim3 grid((unsigned)std::min<int64_t>((L.M + 255) / 256, 64), (unsigned)gn);
      init_master_kernel<<<grid, 256, 0, st>>>(d->w_start, reinterpret_cast<const int*>(stage + rb), gn, L.M, w_out,
                                               d->ldw);
      if (int rc = check_launch("wide init")) return rc;
      convert_kernel<<<dim3(128, (unsigned)gn), 256, 0, st>>>(ca, reinterpret_cast<const StepRow*>(stage), gn);
      if (int rc = check_launch("wide convert")) return rc;
    }
    int t_end = 0;
    for (int i = 0; i < gn; ++i) t_end = std::max(t_end, s1[g0 + i]);
    int t_begin = t_end;
    for (int i = 0; i < gn; ++i) t_begin = std::min(t_begin, s0[g0 + i]);
    for (int t = t_begin; t < t_end; ++t) {
      std::vector<StepRow> rows;
      int max_rows = 1;
      for (int i = 0; i < gn; ++i) {
        const int r = g0 + i;
        if (t < s0[r] || t >= s1[r]) continue;
        const int spe = (nr[r] + bt[r] - 1) / bt[r];
        StepRow sr;
        sr.req = r;
        sr.slot = i;
        sr.e = t / spe;
        sr.s = t % spe;
        sr.rows = std::min(bt[r], nr[r] - sr.s * bt[r]);
        sr.global_step = t;
        sr.lr = (float)lr[(size_t)r * std::max(d->epochs, 1) + sr.e];
        rows.push_back(sr);
        max_rows = std::max(max_rows, sr.rows);
      }
      const int A = (int)rows.size();
      if (A == 0) continue;
      const int nrow = (max_rows + 7) / 8 * 8;  // GEMM row extent of this step
      // pointer arrays: fwd (A, B, C) per layer, bwd per layer, update per layer
      std::vector<const void*> ptrs;
      auto sb = [&](int a) { return slots + (size_t)rows[a].slot * g.slot_bytes; };
      auto wb = [&](int a, int l) { return (const void*)(reinterpret_cast<__nv_bfloat16*>(sb(a)) + g.wb_off[l]); };
      auto act = [&](int a, int l) {  // H_l (l = 0: X)
        return (const void*)(l == 0 ? sb(a) + g.x_off : sb(a) + g.h_off[l]);
      };
      auto dlt = [&](int a, int l) { return (const void*)(sb(a) + g.d_off[l]); };
      auto tmp = [&](int a) { return (const void*)(sb(a) + g.t_off); };
      auto mst = [&](int a, int l) { return (const void*)(w_out + (int64_t)rows[a].req * d->ldw + L.woff[l]); };
      const size_t rows_bytes = (sizeof(StepRow) * A + 255) / 256 * 256;
      // offsets (in pointers) of each array block
      std::vector<size_t> fwdA(H), fwdB(H), fwdC(H), bwdA(H), bwdB(H), bwdC(H), updA(H), updB(H), updC(H);
      auto block = [&](auto fn) {
        const size_t at = ptrs.size();
        for (int a = 0; a < A; ++a) ptrs.push_back(fn(a));
        return at;
      };
      for (int l = 0; l < H; ++l) {
        fwdA[l] = block([&](int a) { return wb(a, l); });
        fwdB[l] = block([&](int a) { return act(a, l); });
        fwdC[l] = block([&](int a) { return tmp(a); });
        updA[l] = block([&](int a) { return dlt(a, l + 1); });
        updB[l] = block([&](int a) { return act(a, l); });
        updC[l] = block([&](int a) { return mst(a, l); });
        if (l >= 1) {
          bwdA[l] = block([&](int a) { return wb(a, l); });
          bwdB[l] = block([&](int a) { return dlt(a, l + 1); });
          bwdC[l] = block([&](int a) { return tmp(a); });
        }
      }
      const size_t stage_need = rows_bytes + ptrs.size() * 8;
      if (stage_need + 256 > d->workspace_bytes - G * g.slot_bytes) {
        set_error("fs_train_bf16 (wide): step staging exceeds the workspace");
        return FS_EINVAL;
      }
      std::vector<uint8_t> host(stage_need);
      memcpy(host.data(), rows.data(), sizeof(StepRow) * A);
      memcpy(host.data() + rows_bytes, ptrs.data(), ptrs.size() * 8);
      cudaMemcpyAsync(stage, host.data(), stage_need, cudaMemcpyHostToDevice, st);
      const StepRow* d_rows = reinterpret_cast<const StepRow*>(stage);
      const void** d_ptrs = reinterpret_cast<const void**>(stage + rows_bytes);
      gather_kernel<<<A, 256, 0, st>>>(sa, d_rows);
      if (int rc = check_launch("wide gather")) return rc;
      // ---- forward
      for (int l = 0; l < H; ++l) {
        const int fin = l == 0 ? g.dp : L.f[l], fout = L.f[l + 1];
        // col-major: Z'(fout x rows) = W'(fout x fin) * H'(fin x rows)
        if (int rc = blas_ok(cublasGemmBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_N, fout, nrow, fin, &one, d_ptrs + fwdA[l],
                                                 CUDA_R_16BF, fout, d_ptrs + fwdB[l], CUDA_R_16BF, fin, &zero,
                                                 (void* const*)(d_ptrs + fwdC[l]), CUDA_R_32F, fout, A,
                                                 CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT),
                             "forward GEMM"))
          return rc;
        fwd_epilogue_kernel<<<dim3((fout + 255) / 256, (unsigned)A), 256, 0, st>>>(sa, d_rows, l + 1);
        if (int rc = check_launch("wide fwd epilogue")) return rc;
      }
      head_kernel<<<A, 256, 0, st>>>(sa, d_rows);
      if (int rc = check_launch("wide head")) return rc;
      // ---- backward: dH_l = D_{l+1} W_l^T (old bf16 weights), then gates
      for (int l = H - 1; l >= 1; --l) {
        const int fin = L.f[l], fout = L.f[l + 1];
        // col-major: dH'(fin x rows) = W'^T (fin x fout) * D'(fout x rows)
        if (int rc = blas_ok(cublasGemmBatchedEx(h, CUBLAS_OP_T, CUBLAS_OP_N, fin, nrow, fout, &one, d_ptrs + bwdA[l],
                                                 CUDA_R_16BF, fout, d_ptrs + bwdB[l], CUDA_R_16BF, fout, &zero,
                                                 (void* const*)(d_ptrs + bwdC[l]), CUDA_R_32F, fin, A,
                                                 CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT),
                             "backward GEMM"))
          return rc;
        gate_kernel<<<dim3((fin + 255) / 256, (unsigned)A), 256, 0, st>>>(sa, d_rows, l);
        if (int rc = check_launch("wide gate")) return rc;
      }
      // ---- updates: W_l master += (-lr) H_l^T D_{l+1}, one batched GEMM per distinct lr
      std::vector<std::pair<float, std::vector<int>>> groups;
      for (int a = 0; a < A; ++a) {
        auto it = std::find_if(groups.begin(), groups.end(), [&](const auto& p) { return p.first == rows[a].lr; });
        if (it == groups.end()) groups.push_back({rows[a].lr, {a}});
        else it->second.push_back(a);
      }
      for (const auto& grp : groups) {
        const float alpha = -grp.first;
        const int ga = (int)grp.second.size();
        const bool contiguous = ga == A;
        for (int l = 0; l < H; ++l) {
          const int fin = l == 0 ? g.dp : L.f[l], fout = L.f[l + 1];
          const int fin_true = L.f[l];  // padded W_0 rows beyond f0 have no master
          const void* const* pa = d_ptrs + updA[l];
          const void* const* pb = d_ptrs + updB[l];
          void* const* pc = (void* const*)(d_ptrs + updC[l]);
          if (!contiguous) {  // sub-batch: gather its pointers into the staging tail
            std::vector<const void*> sub;
            for (size_t blk : {updA[l], updB[l], updC[l]})
              for (int a : grp.second) sub.push_back(ptrs[blk + a]);
            const size_t off = stage_need + 256 + (size_t)3 * A * 8 * l;
            if (off + sub.size() * 8 > d->workspace_bytes - G * g.slot_bytes) {
              set_error("fs_train_bf16 (wide): lr-group staging exceeds the workspace");
              return FS_EINVAL;
            }
            cudaMemcpyAsync(stage + off, sub.data(), sub.size() * 8, cudaMemcpyHostToDevice, st);
            const void** dp = reinterpret_cast<const void**>(stage + off);
            pa = dp;
            pb = dp + ga;
            pc = (void* const*)(dp + 2 * ga);
          }
          (void)fin;
          // col-major: W'(fout x fin) += alpha * D'(fout x rows) * H'^T(rows x fin)
          if (int rc = blas_ok(cublasGemmBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_T, fout, fin_true, nrow, &alpha, pa,
                                                   CUDA_R_16BF, fout, pb, CUDA_R_16BF, l == 0 ? g.dp : L.f[l], &one,
                                                   pc, CUDA_R_32F, fout, ga, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT),
                               "update GEMM"))
            return rc;
        }
      }
      // bf16 copies of the updated masters for the next step
      convert_kernel<<<dim3(128, (unsigned)A), 256, 0, st>>>(ca, d_rows, A);
      if (int rc = check_launch("wide convert")) return rc;
    }
  }
  return FS_OK;
}


// ------------------------------------------------------------------ eval forward (wide layers)
namespace wide {

__global__ void to_bf16_kernel(const float* src, int64_t rows_src, int64_t rows_dst, int cols, __nv_bfloat16* dst) {
  const int64_t total = rows_dst * cols;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += (int64_t)gridDim.x * blockDim.x)
    dst[j] = __float2bfloat16_rn(j / cols < rows_src ? src[j] : 0.f);
}

// H = bf16(relu(Z + b)); the last hidden layer also accumulates the logits
// from the fp32 values (z[r] += sum_u v * w_h[u]), as the trainers do
__global__ void eval_epilogue_kernel(const float* Z, const float* b, int N, int rows, __nv_bfloat16* H,
                                     const float* wh, float* z) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  float v = 0.f;
  if (u < N) {
    v = fmaxf(Z[(int64_t)r * N + u] + b[u], 0.f);
    H[(int64_t)r * N + u] = __float2bfloat16_rn(v);
  }
  if (wh) {
    float p = u < N ? v * wh[u] : 0.f;
    for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
    if ((threadIdx.x & 31) == 0) z[(int64_t)r * zparts(N) + blockIdx.x * 8 + (threadIdx.x >> 5)] = p;
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

}  // namespace wide
}  // namespace fs

using namespace fs;

extern "C" size_t fs_forward_wide_workspace_bytes(const int32_t* dims, int32_t n_dims, int32_t rows) {
  MlpLayout L;
  if (make_layout(dims, n_dims, &L) != FS_OK || rows < 0) return 0;
  const int dp = (L.f[0] + 15) / 16 * 16;
  const size_t wb = ((size_t)L.M + (size_t)(dp - L.f[0]) * L.f[1]) * 2;
  const size_t act = (size_t)rows * std::max(L.max_hidden, dp) * 2;
  return (wb + 255) / 256 * 256 + 2 * ((act + 255) / 256 * 256) +
         (((size_t)rows * L.max_hidden * 4 + 255) / 256 * 256) +
         ((size_t)rows * wide::zparts(L.f[L.L - 1]) * 4 + 256);
}

// K8 forward for layer shapes beyond the on-chip kernels (bf16 operands,
// fp32 accumulation, fp32 head): probs_out[rows] of fs_prep_features_bf16 rows.
extern "C" int fs_forward_wide(const int32_t* dims, int32_t n_dims, const float* w, const void* x_bf16, int32_t rows,
                               double* probs_out, void* workspace, size_t workspace_bytes, void* stream) {
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
  cublasHandle_t h = wide::blas();
  if (!h) {
    set_error("fs_forward_wide: cublasCreate failed");
    return FS_ECUDA;
  }
  if (int rc = wide::blas_ok(cublasSetStream(h, st), "cublasSetStream")) return rc;
  const int dp = (L.f[0] + 15) / 16 * 16;
  uint8_t* p = reinterpret_cast<uint8_t*>(workspace);
  const size_t wb_bytes = ((size_t)L.M + (size_t)(dp - L.f[0]) * L.f[1]) * 2;
  __nv_bfloat16* wb = reinterpret_cast<__nv_bfloat16*>(p);
  p += (wb_bytes + 255) / 256 * 256;
  const size_t act = (size_t)rows * std::max(L.max_hidden, dp) * 2;
  __nv_bfloat16* hbuf[2] = {reinterpret_cast<__nv_bfloat16*>(p),
                            reinterpret_cast<__nv_bfloat16*>(p + (act + 255) / 256 * 256)};
  p += 2 * ((act + 255) / 256 * 256);
  float* Z = reinterpret_cast<float*>(p);
  p += ((size_t)rows * L.max_hidden * 4 + 255) / 256 * 256;
  float* z = reinterpret_cast<float*>(p);  // head-logit partials [rows x zparts]
  const float one = 1.f, zero = 0.f;
  const __nv_bfloat16* in = reinterpret_cast<const __nv_bfloat16*>(x_bf16);
  int fin_pad = dp;
  int64_t wofs = 0;
  for (int l = 0; l < L.L - 1; ++l) {
    const int fin = L.f[l], fout = L.f[l + 1];
    const int kin = l == 0 ? dp : fin;
    __nv_bfloat16* wl = wb + wofs;
    wide::to_bf16_kernel<<<256, 256, 0, st>>>(w + L.woff[l], fin, kin, fout, wl);
    if (int rc = check_launch("fs_forward_wide convert")) return rc;
    wofs += (int64_t)kin * fout;
    // col-major: Z'(fout x rows) = W'(fout x kin) * H'(kin x rows)
    if (int rc = wide::blas_ok(cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, fout, rows, kin, &one, wl, CUDA_R_16BF, fout,
                                            in, CUDA_R_16BF, kin, &zero, Z, CUDA_R_32F, fout, CUBLAS_COMPUTE_32F,
                                            CUBLAS_GEMM_DEFAULT),
                               "forward GEMM"))
      return rc;
    __nv_bfloat16* out = hbuf[l & 1];
    const bool last = l == L.L - 2;
    wide::eval_epilogue_kernel<<<dim3((fout + 255) / 256, (unsigned)rows), 256, 0, st>>>(
        Z, w + L.boff[l], fout, rows, out, last ? w + L.woff[L.L - 1] : nullptr, z);
    if (int rc = check_launch("fs_forward_wide epilogue")) return rc;
    in = out;
    fin_pad = fout;
  }
  (void)fin_pad;
  wide::eval_probs_kernel<<<(rows + 255) / 256, 256, 0, st>>>(z, wide::zparts(L.f[L.L - 1]), w + L.boff[L.L - 1],
                                                              rows, probs_out);
  return check_launch("fs_forward_wide probs");
}

