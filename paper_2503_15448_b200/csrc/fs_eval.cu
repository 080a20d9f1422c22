// K8 metrics half: accuracy and rank AUC of the per-round evaluation.
//
// Replaces metrics.evaluate / accuracy / auc_roc / _midranks
// (pkg/src/fedsim/metrics.py:118-165), run every round by
// FederationEngine._emit_report (server.py:321-353).  The eval forward
// itself is fs_forward_f64 (K8 forward half, fs_train_f64.cu).
//
// AUC = U_pos / (n_pos * n_neg) with U_pos = sum over positives of
// (#negatives scoring below + 0.5 * #negatives tied) — the midrank
// identity.  Everything is counted in integers (2*U exactly), so the
// result equals the reference's midrank sum bit for bit given equal scores.
#include <cub/device/device_radix_sort.cuh>

#include "fs_common.cuh"

namespace fs {

template <typename K>
__device__ __forceinline__ K key_inf();
template <>
__device__ __forceinline__ double key_inf<double>() { return __longlong_as_double(0x7ff0000000000000LL); }
template <>
__device__ __forceinline__ float key_inf<float>() { return __int_as_float(0x7f800000); }

// counts: [0]=correct, [1]=2U, [2]=n_pos, [3]=n_neg
// K = float when every score is a widened float (the bf16 evaluation): the
// keys convert exactly and the radix sort needs 4 digit passes instead of 8
template <typename K>
__global__ void eval_split_kernel(const double* scores, const int8_t* labels, int n, double thr,
                                  K* neg_keys, unsigned long long* counts) {
  unsigned correct = 0, pos = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double s = scores[i];
    const bool is_pos = labels[i] == 1;
    correct += ((s >= thr) == is_pos);
    pos += is_pos;
    neg_keys[i] = is_pos ? key_inf<K>() : (K)s;  // +inf sorts last
  }
  correct = __reduce_add_sync(0xffffffffu, correct);
  pos = __reduce_add_sync(0xffffffffu, pos);
  if ((threadIdx.x & 31) == 0) {
    if (correct) atomicAdd(counts + 0, (unsigned long long)correct);
    if (pos) atomicAdd(counts + 2, (unsigned long long)pos);
  }
}

template <typename K>
__global__ void eval_rank_kernel(const double* scores, const int8_t* labels, int n,
                                 const K* sorted_neg, unsigned long long* counts) {
  const int n_neg = n - (int)counts[2];
  unsigned long long twice_u = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (labels[i] != 1) continue;
    const K s = (K)scores[i];
    int lo = 0, hi = n_neg;  // first index with key >= s
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sorted_neg[mid] < s) lo = mid + 1; else hi = mid;
    }
    int lo2 = lo, hi2 = n_neg;  // first index with key > s
    while (lo2 < hi2) {
      const int mid = (lo2 + hi2) >> 1;
      if (sorted_neg[mid] <= s) lo2 = mid + 1; else hi2 = mid;
    }
    twice_u += 2ull * (unsigned long long)lo + (unsigned long long)(lo2 - lo);
  }
  for (int o = 16; o > 0; o >>= 1) twice_u += __shfl_xor_sync(0xffffffffu, twice_u, o);
  if ((threadIdx.x & 31) == 0 && twice_u) atomicAdd(counts + 1, twice_u);
}

template <typename K>
static size_t cub_temp_bytes(int n) {
  size_t t = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, t, (const K*)nullptr, (K*)nullptr, n);
  return t;
}

template <typename K>
static int eval_metrics(const double* scores, const int8_t* labels, int32_t n, double threshold,
                        int64_t* counts_out, char* ws, cudaStream_t st) {
  auto* counts = reinterpret_cast<unsigned long long*>(ws);
  K* keys = reinterpret_cast<K*>(ws + 256);
  K* sorted = keys + ((size_t)n + 31) / 32 * 32;
  void* temp = reinterpret_cast<void*>(sorted + ((size_t)n + 31) / 32 * 32);
  size_t temp_bytes = cub_temp_bytes<K>(n);
  if (cudaMemsetAsync(counts, 0, 4 * sizeof(unsigned long long), st) != cudaSuccess)
    return check_launch("memset counts");
  int blocks = (n + 255) / 256;
  if (blocks > 4 * kNumSMs) blocks = 4 * kNumSMs;
  eval_split_kernel<K><<<blocks, 256, 0, st>>>(scores, labels, n, threshold, keys, counts);
  if (int rc = check_launch("eval_split_kernel")) return rc;
  if (cub::DeviceRadixSort::SortKeys(temp, temp_bytes, keys, sorted, n, 0, (int)(8 * sizeof(K)), st) !=
      cudaSuccess)
    return check_launch("cub sort");
  eval_rank_kernel<K><<<blocks, 256, 0, st>>>(scores, labels, n, sorted, counts);
  if (int rc = check_launch("eval_rank_kernel")) return rc;
  if (cudaMemcpyAsync(counts_out, counts, 3 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return check_launch("copy counts");
  return FS_OK;
}

}  // namespace fs

using namespace fs;

extern "C" size_t fs_eval_workspace_bytes(int32_t n) {
  if (n < 1) return 0;
  const size_t padded = ((size_t)n + 31) / 32 * 32;
  return 256 + 2 * padded * sizeof(double) + cub_temp_bytes<double>(n) + 256;
}

extern "C" int fs_eval_metrics(const double* scores, const int8_t* labels, int32_t n,
                               double threshold, int64_t* counts_out, void* workspace,
                               size_t workspace_bytes, void* stream) {
  if (n < 1 || workspace_bytes < fs_eval_workspace_bytes(n)) {
    set_error("fs_eval_metrics: empty input or workspace too small");
    return FS_EINVAL;
  }
  return eval_metrics<double>(scores, labels, n, threshold, counts_out, reinterpret_cast<char*>(workspace),
                              (cudaStream_t)stream);
}

extern "C" int fs_eval_metrics_f32(const double* scores, const int8_t* labels, int32_t n,
                                   double threshold, int64_t* counts_out, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  if (n < 1 || workspace_bytes < fs_eval_workspace_bytes(n)) {
    set_error("fs_eval_metrics_f32: empty input or workspace too small");
    return FS_EINVAL;
  }
  if (cub_temp_bytes<float>(n) > cub_temp_bytes<double>(n)) {
    set_error("fs_eval_metrics_f32: sort workspace");
    return FS_EINVAL;
  }
  return eval_metrics<float>(scores, labels, n, threshold, counts_out, reinterpret_cast<char*>(workspace),
                             (cudaStream_t)stream);
}
