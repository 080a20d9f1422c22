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

// Packs keep-bits of one stream: bit j = (random_j < keep). Each thread
// jumps its own PCG64 copy ahead to its first word and steps sequentially.
// random() = (x >> 11) * 2^-53 < keep  <=>  (x >> 11) < ceil(keep * 2^53),
// so the comparison runs on integers (threshold computed exactly on host).
__device__ void mask_stream(const Pcg64& base, int64_t n_draws, uint64_t thresh, uint32_t* out) {
  const int64_t words = (n_draws + 31) / 32;
  const int64_t wpt = (words + MASK_THREADS - 1) / MASK_THREADS;
  const int64_t w0 = threadIdx.x * wpt;
  const int64_t w1 = min(words, w0 + wpt);
  if (w0 >= w1) return;
  Pcg64 g = base;
  g.advance((uint64_t)(w0 * 32));
  for (int64_t w = w0; w < w1; ++w) {
    uint32_t bits = 0;
    const int64_t lim = min((int64_t)32, n_draws - w * 32);
    if (lim == 32) {
#pragma unroll 8
      for (int b = 0; b < 32; ++b) bits |= (uint32_t)((g.next64() >> 11) < thresh) << b;
    } else {
      for (int b = 0; b < lim; ++b) bits |= (uint32_t)((g.next64() >> 11) < thresh) << b;
    }
    out[w] = bits;
  }
}

__global__ void __launch_bounds__(MASK_THREADS)
    dropout_bits_kernel(const uint64_t* seeds, const int32_t* n_rows, const int32_t* batch,
                        const int64_t* mask_off, int epochs, int sum_hidden, uint64_t thresh,
                        uint32_t* bits) {
  const int r = blockIdx.x;
  const int n = n_rows[r], B = batch[r];
  const int spe = (n + B - 1) / B;
  const int64_t slot = ((int64_t)B * sum_hidden + 31) / 32;
  const uint64_t train_seed = seeds[r];
  for (int st = blockIdx.y; st < epochs * spe; st += gridDim.y) {
    const int e = st / spe, s = st % spe;
    const int rows = min(B, n - s * B);
    const Pcg64 base = pcg_from_seed(derive_mask_seed(train_seed, (uint32_t)e, (uint32_t)s));
    mask_stream(base, (int64_t)rows * sum_hidden, thresh, bits + mask_off[r] + (int64_t)st * slot);
  }
}

__global__ void __launch_bounds__(MASK_THREADS)
    dropout_bits_seed_kernel(uint64_t mask_seed, int64_t n_draws, uint64_t thresh, uint32_t* bits) {
  mask_stream(pcg_from_seed(mask_seed), n_draws, thresh, bits);
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
  const size_t smem = (size_t)max_rows * sizeof(int32_t);
  const int use_smem = smem <= 200 * 1024;
  if (use_smem && smem > 48 * 1024)
    cudaFuncSetAttribute(shuffle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  shuffle_kernel<<<n_req * epochs, 128, use_smem ? smem : 0, (cudaStream_t)stream>>>(
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
  dim3 grid(n_req, MASK_YSPLIT);
  dropout_bits_kernel<<<grid, MASK_THREADS, 0, (cudaStream_t)stream>>>(
      seeds, n_rows, batch, mask_off, epochs, sum_hidden, keep_threshold(keep), bits_out);
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
